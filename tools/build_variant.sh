#!/bin/bash
# build the engine with extra nvcc defines for mine_general.cu into OUT.so
# usage: tools/build_variant.sh OUT.so -DFOO=1 ...
out=$1; shift
B=paper_1208_4271_b200; mkdir -p /tmp/bv
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC -I include "$@" -c $B/csrc/mine_general.cu -o /tmp/bv/mine_general.cu.o
objs=$(ls build/*.o | grep -v mine_general.cu.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $out $objs /tmp/bv/mine_general.cu.o -lpthread
