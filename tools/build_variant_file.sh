#!/bin/bash
# build a variant of libtempokkt_b200.so with extra -D flags for ONE source file
# usage: tools/build_variant_file.sh <file.cu> <name> <flags...>   -> paper_2405_04808_b200/lib_<name>.so
set -e
f=$1; name=$2; shift; shift
P=paper_2405_04808_b200
B=$P/_build
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -I include -I $P/csrc "$@" \
  -c $P/csrc/$f -o /tmp/var_$name.o
objs=$(ls $B/*.o | grep -v "/$f.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $P/lib_$name.so $objs /tmp/var_$name.o -lcudart
echo built $P/lib_$name.so
