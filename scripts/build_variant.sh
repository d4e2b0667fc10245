#!/bin/bash
# Build libmrfp4.so with extra -D flags on one source (VSRC, default gemm_fp4) into
# build/var_<name>/ (perf experiments; load with MRFP4_LIB=build/var_<name>/libmrfp4.so).
# Usage: [VSRC=linear_decode] scripts/build_variant.sh <name> <flags...>
name=$1; shift
src=${VSRC:-gemm_fp4}
set -e
make -s -j8 >/dev/null
mkdir -p build/var_$name
nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-O3 -Xptxas -O3 \
  --expt-relaxed-constexpr "$@" -c paper_2509_23202_b200/csrc/$src.cu -o build/var_$name/$src.o
objs=$(ls build/obj/*.o | grep -v "/$src.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/var_$name/libmrfp4.so build/var_$name/$src.o $objs -lcuda
echo built build/var_$name/libmrfp4.so
