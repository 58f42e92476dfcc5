#!/bin/bash
# usage: tools/ncu_top.sh <kernel-regex> <out-name> [launch-skip]
# one --set full capture of the first matching launch of a V-cycle (configs[2])
k=$1; o=$2; s=${3:-0}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$k" -s $s -c 1 \
  -o gpurun_out/$o python tools/prof_vcycle.py 2 1 > gpurun_out/$o.log 2>&1
echo "ncu rc=$?"
