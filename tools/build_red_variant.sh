#!/bin/bash
# Library variant with extra flags for the reduction translation unit only:
#   bash tools/build_red_variant.sh NAME "-DGT_RED_UNROLL=8"  -> build_vNAME/libglucosim.so
set -e
cd "$(dirname "$0")/.."
make -C paper_2202_13927_b200/csrc -s
name=$1; shift
mkdir -p build_v$name
C=paper_2202_13927_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --fmad=true $@ \
  -c $C/gt_reduce.cu -o build_v$name/gt_reduce.o 2> build_v$name/ptxas.txt
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build_v$name/libglucosim.so \
  $C/build/gt_parity.o $C/build/gt_sampler.o $C/build/gt_fast.o build_v$name/gt_reduce.o $C/build/gt_northern.o \
  $C/build/gt_capi.o -lcudart
echo "built build_v$name"
