o=gpurun_out/s23_ab.log; rm -f $o
for rep in 1 2; do
  for spec in "base:X=1" "gsb64:HPG_LIB=abtmp/gsb64.so" "low128:HPG_LIB=abtmp/low128.so" "spmv128:HPG_LIB=abtmp/spmv128.so"; do
    label=${spec%%:*}; envs=${spec#*:}
    env $envs timeout 300 python tools/microbench.py --brief "$label" 2>&1 | tail -1 >> $o
  done
done
cat $o
