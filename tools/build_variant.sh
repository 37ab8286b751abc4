#!/bin/bash
# Build a K1 experiment variant of the library: tools/build_variant.sh NAME -DFLAG=V ...
# -> paper_1509_08360_b200/libcsemb_cuda_NAME.so (csemb_cuda.cu recompiled with the
# flags, the other translation units reused from build/csemb_obj).  Select it at
# run time with CSEMB_LIB_PATH.  Experiments only; never the shipped library.
set -e
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
NAME=$1; shift
OBJ=$ROOT/build/csemb_obj
python -c "import sys; sys.path.insert(0, '$ROOT'); from paper_1509_08360_b200.build import build; build(verbose=False)"
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC "$@" \
    -c -o $OBJ/csemb_cuda_$NAME.o $ROOT/paper_1509_08360_b200/csrc/csemb_cuda.cu
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o $ROOT/paper_1509_08360_b200/libcsemb_cuda_$NAME.so \
    $OBJ/csemb_cuda_$NAME.o $OBJ/downstream.cu.o $OBJ/build.cu.o $OBJ/diag.cu.o
echo "built libcsemb_cuda_$NAME.so ($*)"
