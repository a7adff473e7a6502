#!/bin/sh
# Build the sm_100a shared library (also done by __graft_entry__.build()).
set -e
cd "$(dirname "$0")"
nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xptxas -v \
     -shared -Xcompiler -fPIC -o paper_1711_11407_b200/libfpssft.so \
     paper_1711_11407_b200/csrc/fpssft.cu "$@"
