timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/s20_gputests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/s20_gputests.log
o=gpurun_out/s20_ab.log; rm -f $o
for rep in 1 2; do
  for spec in "base:X=1" "st0:HPG_STENCIL=0" "nomagic:HPG_LIB=abtmp/nomagic.so" "spmv3:HPG_LIB=abtmp/spmv3.so" "minb4:HPG_GS_MINB=4"; do
    label=${spec%%:*}; envs=${spec#*:}
    env $envs timeout 300 python tools/microbench.py --brief "$label" 2>&1 | tail -1 >> $o
  done
done
cat $o
