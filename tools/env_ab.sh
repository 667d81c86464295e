#!/bin/bash
# Same-box A/B over environment settings of the in-tree build:
#   tools/env_ab.sh OUTLOG "label:VAR=val VAR2=val" ...   (two interleaved rounds)
out=$1; shift
for rep in 1 2; do
  for spec in "$@"; do
    label=${spec%%:*}; envs=${spec#*:}
    env $envs timeout 300 python tools/microbench.py --brief "$label" 2>&1 | tail -1 >> "$out"
  done
done
