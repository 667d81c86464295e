#!/bin/bash
# One profiling pass on the GPU box (run from the repo root under gpurun):
#   1. the bench line (no profiler)
#   2. ncu launch list of one 30-iteration restart cycle of the timed solve
#   3. ncu --set full of the hot kernels (one launch each kind)
# Outputs land in gpurun_out/<tag>_*.
tag=${1:-prof}
NCU=${NCU:-ncu}
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench rc=$?"
timeout 900 $NCU --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
  python tools/profile_solve.py --iters 30 > gpurun_out/${tag}_launches.log 2>&1
echo "launches rc=$?"
timeout 900 $NCU --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:'k_gs_pass|k_gs_lower|k_spmv|k_cgs2_fused|k_restrict' -c 12 -f -o gpurun_out/${tag}_full \
  python tools/prof_parts.py > gpurun_out/${tag}_full.log 2>&1
echo "full rc=$?"
