#!/bin/bash
# usage: tools/build_variant.sh OUT.so [-DFOO ...] -- experiment / instrumented builds of libsten (tools only)
out=$1; shift
cd "$(dirname "$0")/../paper_2304_07613_b200" && /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -shared --split-compile=0 --expt-relaxed-constexpr -Xptxas -warn-spills "$@" -I ../include -I csrc \
  -o "$out" csrc/*.cu
