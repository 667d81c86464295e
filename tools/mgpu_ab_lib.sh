#!/bin/bash
# Multi-GPU A/B over (library build, environment): tools/mgpu_ab_lib.sh N TAG "label:lib:VAR=val ..." ...
n=$1; tag=$2; shift 2
port=29700
for rep in 1 2; do
  for spec in "$@"; do
    label=${spec%%:*}; rest=${spec#*:}; lib=${rest%%:*}; envs=${rest#*:}; port=$((port+1))
    if [ "$lib" = base ]; then libp=""; else libp=$PWD/abtmp/$lib.so; fi
    env HPG_LIB=$libp $envs timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
      --master-addr 127.0.0.1 --master-port $port bench.py --gpus $n --steps 3 --warmup 3 --no-validation --no-cpu \
      2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$label', round(d['value'],1), round(d['ms_per_step'],1), round(d['fp64_gflops'],1))" >> gpurun_out/${tag}_bench.log
  done
done
