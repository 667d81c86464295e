#!/bin/bash
# Same-box A/B of library variants built by tools/build_variant.sh:
#   tools/ab_run.sh OUTLOG base variant1 variant2 ...   (base = the in-tree build)
out=$1; shift
for rep in 1 2; do
  for v in "$@"; do
    if [ "$v" = base ]; then lib=""; else lib=abtmp/$v.so; fi
    HPG_LIB=$lib timeout 300 python tools/microbench.py --brief "$v" 2>&1 | tail -1 >> "$out"
  done
done
