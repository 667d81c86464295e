timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s21_gputests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/s21_gputests.log
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > gpurun_out/s21_bench1.json 2> gpurun_out/s21_bench1.err; echo "bench1 rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 > gpurun_out/s21_bench2.json 2> gpurun_out/s21_bench2.err; echo "bench2 rc=$?"
