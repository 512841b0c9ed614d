#!/bin/bash
# Builds build_var/lib_<name>.so with extra nvcc flags (probe with EMRKC_LIB).
# Usage: tools/build_variant.sh <name> [nvcc flags...]
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p build_var
S=paper_2401_01745_b200/csrc
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 \
  -Xcompiler -fPIC -Xcompiler -O2 -shared "$@" -o build_var/lib_$name.so \
  $S/kernels.cu $S/kernels_fast.cu $S/emrkc_generic.cu $S/emrkc_capi.cpp
