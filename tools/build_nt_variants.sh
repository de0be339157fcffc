#!/bin/bash
# Developer: build libpolyjac_b200 variants differing only in newton.cu compile flags into tools/_exp/
# usage: bash tools/build_nt_variants.sh "NAME:-DFLAG=1 -DFLAG2=3" ...
set -e
cd "$(dirname "$0")/.."
B=paper_1201_0499_b200/_build
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-ffp-contract=off -fmad=false \
      $flags -c paper_1201_0499_b200/csrc/newton.cu -o tools/_exp/newton_$name.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/_exp/lib_$name.so $B/eval_kernels.cu.o $B/eval_fast.cu.o $B/eval_fastd.cu.o \
      tools/_exp/newton_$name.o $B/fp64_probe.cu.o $B/capi.cpp.o $B/sysio.cpp.o -Xlinker --version-script=$B/exports.map
  echo built $name
done
