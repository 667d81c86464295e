timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s25_gputests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/s25_gputests.log
timeout 300 python tools/microbench.py --brief wave_st > gpurun_out/s25_mb.log 2>&1; tail -1 gpurun_out/s25_mb.log
HPG_STENCIL=0 timeout 300 python tools/microbench.py --brief st0 >> gpurun_out/s25_mb.log 2>&1; tail -1 gpurun_out/s25_mb.log
timeout 600 python bench.py > gpurun_out/s25_bench1.json 2> gpurun_out/s25_bench1.err; echo "bench1 rc=$?"
