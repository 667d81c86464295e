#!/bin/bash
# Multi-GPU A/B of environment settings (torchrun, N ranks): bench lines and
# comm latencies.  tools/mgpu_ab.sh N OUTTAG "label:VAR=val ..." ...
n=$1; tag=$2; shift 2
port=29600
for rep in 1 2; do
  for spec in "$@"; do
    label=${spec%%:*}; envs=${spec#*:}; port=$((port+1))
    env $envs timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $port bench.py --gpus $n --steps 3 --warmup 3 --no-validation --no-cpu 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$label', round(d['value'],1), round(d['ms_per_step'],1), round(d['fp64_gflops'],1))" >> gpurun_out/${tag}_bench.log
  done
done
for spec in "$@"; do
  label=${spec%%:*}; envs=${spec#*:}; port=$((port+1))
  env $envs timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $port tools/mgpu_comm.py 256 2>/dev/null | grep '"rank": 0' | sed "s/^/$label /" >> gpurun_out/${tag}_comm.log
done
