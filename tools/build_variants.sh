#!/bin/bash
# Developer A/B: build libpolyjac_b200 variants that differ only in one source file's compile flags.
# usage: bash tools/build_variants.sh FILE.cu "NAME:-DFLAG=1 -DFLAG2=3" ...   -> tools/_exp/lib_NAME.so
# (the other objects come from paper_1201_0499_b200/_build; run the normal build first)
set -e
cd "$(dirname "$0")/.."
B=paper_1201_0499_b200/_build
F=$1; shift
mkdir -p tools/_exp
objs=""
for o in eval_kernels.cu eval_fast.cu eval_fast_ws.cu eval_fastd.cu newton.cu fp64_probe.cu capi.cpp sysio.cpp; do
  [ "$o" = "$F" ] || objs="$objs $B/$o.o"
done
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-ffp-contract=off -fmad=false \
      $flags -c paper_1201_0499_b200/csrc/$F -o tools/_exp/${F%.cu}_$name.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/_exp/lib_$name.so $objs tools/_exp/${F%.cu}_$name.o \
      -Xlinker --version-script=$B/exports.map
  rm -f tools/_exp/${F%.cu}_$name.o
  echo built $name
done
