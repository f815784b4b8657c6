#!/bin/bash
# build the engine with extra nvcc defines for one kernel source into OUT.so
# usage: [SRC=mine_kernels.cu] tools/build_variant.sh OUT.so -DFOO=1 ...
out=$1; shift
src=${SRC:-mine_general.cu}
B=paper_1208_4271_b200; BV=/tmp/bv/$(basename $out .so); mkdir -p $BV
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC -I include -I build/gen "$@" -c $B/csrc/$src -o $BV/$src.o
objs=$(ls build/*.o | grep -v "$src.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $out $objs $BV/$src.o -lpthread -ldl
