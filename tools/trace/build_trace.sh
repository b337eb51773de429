#!/bin/bash
# scratch build of the library with k_final phase tracing (-DTPB_TRACE)
set -e
cd "$(dirname "$0")"; mkdir -p ../../scratch/trace_lib

C=../../paper_2510_27351_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -DTPB_TRACE -c $C/tp_kernels.cu -o ../../scratch/trace_lib/tp_kernels.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../scratch/trace_lib/libtridpart_b200.so ../../scratch/trace_lib/tp_kernels.o ../../paper_2510_27351_b200/lib/tp_capi.o ../../paper_2510_27351_b200/lib/tp_knn.o -cudart static
