#!/bin/bash
# Build libmrfp4.so with extra -D flags on gemm_fp4.cu into build/var_<name>/ (perf experiments;
# load with MRFP4_LIB=build/var_<name>/libmrfp4.so).  Usage: scripts/build_variant.sh <name> <flags...>
name=$1; shift
set -e
make -s -j8 >/dev/null
mkdir -p build/var_$name
nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-O3 -Xptxas -O3 \
  --expt-relaxed-constexpr "$@" -c paper_2509_23202_b200/csrc/gemm_fp4.cu -o build/var_$name/gemm_fp4.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/var_$name/libmrfp4.so build/var_$name/gemm_fp4.o \
  build/obj/act_quant.o build/obj/capi.o build/obj/mse_search.o build/obj/sf_layout.o -lcuda
echo built build/var_$name/libmrfp4.so
