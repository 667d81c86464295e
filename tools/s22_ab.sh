o=gpurun_out/s22_ab.log; rm -f $o
for rep in 1 2; do
  for spec in "base:X=1" "l2hint:HPG_LIB=abtmp/l2hint.so" "gsb128:HPG_LIB=abtmp/gsb128.so" "gsb512:HPG_LIB=abtmp/gsb512.so"; do
    label=${spec%%:*}; envs=${spec#*:}
    env $envs timeout 300 python tools/microbench.py --brief "$label" 2>&1 | tail -1 >> $o
  done
done
cat $o
