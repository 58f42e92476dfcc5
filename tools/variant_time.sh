#!/bin/bash
# time the fine Jacobi sweep of configs[2] for the default library and variants: tools/variant_time.sh v1 v2 ...
for v in default "$@" default "$@"; do
  if [ $v = default ]; then L=paper_2405_04808_b200/libtempokkt_b200.so; else L=paper_2405_04808_b200/lib_$v.so; fi
  TK_LIB_PATH=$L timeout 300 python tools/time_jacobi.py 2 $v 2>&1 | tail -1
done
