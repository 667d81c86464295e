timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s24_gputests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/s24_gputests.log
timeout 600 python bench.py > gpurun_out/s24_bench1.json 2> gpurun_out/s24_bench1.err; echo "bench1 rc=$?"
tools/profile_one.sh r01g k_gs_pass 16 2
tools/profile_one.sh r01g k_gs_lower_st 1 2
tools/profile_one.sh r01g k_spmv 0 2
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01g_bench_launches.csv \
  python bench.py --steps 1 --warmup 1 --max-iters 30 --no-validation --no-cpu > gpurun_out/r01g_bench_launches.log 2>&1
echo "launches rc=$?"
python tools/summarize_ncu.py --launches gpurun_out/r01g_bench_launches.csv > gpurun_out/r01g_bench_launches.md 2>&1
gzip -f gpurun_out/r01g_bench_launches.csv
du -sh gpurun_out
