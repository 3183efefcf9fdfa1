#!/bin/bash
# Build an A/B variant of libfht.so: tools/build_variant.sh NAME "-DFHT_X=0 ..." -> build/ab/NAME.so
set -e
cd "$(dirname "$0")/.."
mkdir -p build/ab
nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC,-O2,-ffp-contract=off -shared \
  -I include $2 -o build/ab/$1.so paper_1811_06378_b200/csrc/fht_api.cu
