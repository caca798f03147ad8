#!/bin/bash
# Build an experiment variant of the library with extra nvcc defines for one
# source, e.g.  tools/build_variant.sh gemm_i8 v1 -DMOE_EPI_VARIANT=1
# -> paper_2508_07329_b200/lib/variants/libmoe_b200_v1.so (load with MOE_B200_LIB=...)
set -e
cd "$(dirname "$0")/.."
src=$1; tag=$2; shift 2
L=paper_2508_07329_b200/lib
mkdir -p $L/variants
python -m paper_2508_07329_b200.build > /dev/null
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr \
  -DNDEBUG "$@" -c paper_2508_07329_b200/csrc/$src.cu -o $L/variants/$src.$tag.o
objs=$(ls $L/obj/*.o | grep -v "/$src.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $L/variants/libmoe_b200_$tag.so $objs $L/variants/$src.$tag.o
echo $L/variants/libmoe_b200_$tag.so
