#!/bin/bash
# Build a profiling / ablation variant of libovx.so into tools/abl/: build_variant.sh NAME NVCC_FLAGS...
#   e.g. tools/build_variant.sh trace -DOVX_TRACE=600
set -e
cd "$(dirname "$0")/../paper_2404_13683_b200/csrc"
name=$1; shift
mkdir -p ../../tools/abl
nvcc -O3 -std=c++17 -shared -Xcompiler -fPIC,-ffp-contract=off -gencode arch=compute_100a,code=sm_100a "$@" \
     -o ../../tools/abl/libovx_$name.so kernels.cu capi.cu element_setup.cpp 2>&1 | grep -i " error" || true
ls -la ../../tools/abl/libovx_$name.so
