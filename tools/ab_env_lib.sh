#!/bin/bash
# Same-box A/B over (library build, environment) pairs, two interleaved rounds:
#   tools/ab_env_lib.sh OUTLOG "label:lib:VAR=val ..." ...   (lib: base | abtmp name)
out=$1; shift
for rep in 1 2; do
  for spec in "$@"; do
    label=${spec%%:*}; rest=${spec#*:}; lib=${rest%%:*}; envs=${rest#*:}
    if [ "$lib" = base ]; then libp=""; else libp=abtmp/$lib.so; fi
    env HPG_LIB=$libp $envs timeout 300 python tools/microbench.py --brief "$label" 2>&1 | tail -1 >> "$out"
  done
done
