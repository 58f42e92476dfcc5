#!/bin/bash
# build a variant of libtempokkt_b200.so with extra -D flags for tk_tri_part.cu only
# usage: tools/build_variant.sh <name> <flags...>   -> paper_2405_04808_b200/lib_<name>.so
set -e
name=$1; shift
P=paper_2405_04808_b200
B=$P/_build
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -I include -I $P/csrc "$@" \
  -c $P/csrc/tk_tri_part.cu -o /tmp/part_$name.o
objs=$(ls $B/*.o | grep -v tk_tri_part)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $P/lib_$name.so $objs /tmp/part_$name.o -lcudart
echo built $P/lib_$name.so
