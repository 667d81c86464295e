#!/bin/bash
# Build libhpgmxp.so with extra nvcc flags into abtmp/<name>.so for same-box A/B
# runs (HPG_LIB=abtmp/<name>.so).  Usage: tools/build_variant.sh NAME -DFLAG=1 ...
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p abtmp
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -shared \
  -I include -I paper_2507_11512_b200/csrc "$@" paper_2507_11512_b200/csrc/*.cu -o abtmp/$name.so -lnccl
echo abtmp/$name.so
