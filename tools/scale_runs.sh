#!/bin/bash
# Weak-scaling and config-4/5 bench lines on one box (run under gpurun --gpus 4).
# Each line lands in gpurun_out/<tag>_<what>.json; bench logs beside it.
tag=${1:-r02}
out=gpurun_out
run() {  # name, nproc, extra args
  local name=$1 np=$2; shift 2
  if [ "$np" = 1 ]; then
    timeout 900 python bench.py "$@" > $out/${tag}_$name.log 2>&1
  else
    CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((np-1))) timeout 900 python -m torch.distributed.run --nnodes=1 \
      --nproc-per-node $np --master-addr 127.0.0.1 --master-port $((29500+np)) bench.py --gpus $np "$@" \
      > $out/${tag}_$name.log 2>&1
  fi
  echo "$name rc $?"
  grep '^{' $out/${tag}_$name.log | tail -n 1 > $out/${tag}_$name.json
}
run bench_1gpu 1 --steps 3 --warmup 3
run bench_2gpu 2 --steps 3 --warmup 3
run bench_4gpu 4 --steps 3 --warmup 3
run bench_1gpu_320 1 --steps 2 --warmup 3 --local 320 --no-cpu
run bench_4gpu_fullscale 4 --steps 2 --warmup 3 --validation fullscale
