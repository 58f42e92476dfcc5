#!/bin/bash
# V-cycle + substitution times of configs[2] for library variants (TK_LIB_PATH):
# usage: tools/lib_ab.sh default v1 v2 ...   (v -> paper_2405_04808_b200/lib_v.so)
for v in "$@"; do
  if [ "$v" = default ]; then unset TK_LIB_PATH; else export TK_LIB_PATH=paper_2405_04808_b200/lib_$v.so; fi
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --solve-config -1 > gpurun_out/l_bench_$v.log 2>gpurun_out/l_bench.err || echo "bench $v failed"
  python3 - "$v" "gpurun_out/l_bench_$v.log" <<'PY'
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().split("\n")[-1])
k = d["kernels"]
print(sys.argv[1], "ms/V-cycle", round(d["ms_per_step"], 3), "fwd", k["tk_forward_subst"]["ms"], k["tk_forward_subst"]["calls"], "back", k["tk_sgs_back_half"]["ms"])
PY
done
