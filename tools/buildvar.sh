#!/bin/bash
# usage: tools/buildvar.sh name "-DFOO=1 -DBAR=2"   -> sweep/lib_<name>.so (variant build)
mkdir -p sweep
cd paper_1308_2144_b200/csrc
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false \
  -Xcompiler -fPIC -Xptxas -v -shared $2 -o ../../sweep/lib_$1.so hyperball.cu 2> ../../sweep/ptxas_$1.log \
  || { tail ../../sweep/ptxas_$1.log; exit 1; }
