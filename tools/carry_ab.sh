#!/bin/bash
# V-cycle + substitution times for carry group sizes / chunk lengths:
# usage: tools/carry_ab.sh "G:Lc" ...   (def = built-in choice)
for spec in "$@"; do
  g=${spec%%:*}; lc=${spec##*:}
  if [ "$g" = def ]; then unset TK_CARRY_GROUP; else export TK_CARRY_GROUP=$g; fi
  if [ "$lc" = def ]; then unset TK_CHAIN_CHUNK; else export TK_CHAIN_CHUNK=$lc; fi
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --solve-config -1 > gpurun_out/g_bench_$g_$lc.log 2>gpurun_out/g_bench.err; echo "bench $spec rc=$?"
  python3 - "$spec" "gpurun_out/g_bench_$g_$lc.log" <<'PY'
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().split("\n")[-1])
k = d["kernels"]
print(sys.argv[1], "ms/V-cycle", round(d["ms_per_step"], 3), "fwd", k["tk_forward_subst"]["ms"], k["tk_forward_subst"]["calls"], "back", k["tk_sgs_back_half"]["ms"])
PY
done
