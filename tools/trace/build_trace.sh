#!/bin/bash
# scratch build of the library with finishing-solve phase tracing (-DTPB_TRACE);
# extra nvcc flags (e.g. -DTPB_LF_STAGE=1) and TRACE_OUT (output dir) are optional
set -e
cd "$(dirname "$0")"
OUT=${TRACE_OUT:-../../scratch/trace_lib}; mkdir -p $OUT
C=../../paper_2510_27351_b200/csrc
L=../../paper_2510_27351_b200/lib
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -DTPB_TRACE "$@" -c $C/tp_kernels.cu -o $OUT/tp_kernels.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libtridpart_b200.so $OUT/tp_kernels.o $L/tp_capi.o $L/tp_knn.o $L/tp_stage.o -cudart static
