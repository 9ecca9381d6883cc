#!/bin/bash
# tools/build_variant.sh NAME [nvcc -D flags...] -> build_variants/NAME.so (kernel A/B experiments)
cd "$(dirname "$0")/.." || exit 1
name=$1; shift
mkdir -p build_variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -lnccl \
  -I include "$@" -o build_variants/$name.so paper_1605_04821_b200/csrc/hjb.cu
