#!/bin/bash
# substitution tests + per-call breakdown of the coarse solve for several chunk lengths
timeout 900 python -m pytest tests/test_gpu_sizes.py tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_gpu_shapes.py -x -q > gpurun_out/c_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/c_tests.log
for lc in "$@"; do
  if [ "$lc" = old ]; then export TK_CHAIN_WARP=0; unset TK_CHAIN_CHUNK; elif [ "$lc" = def ]; then unset TK_CHAIN_WARP; unset TK_CHAIN_CHUNK; else unset TK_CHAIN_WARP; export TK_CHAIN_CHUNK=$lc; fi
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --solve-config -1 > gpurun_out/c_bench_$lc.log 2>gpurun_out/c_bench_$lc.err; echo "bench $lc rc=$?"
  python3 - "$lc" <<'PY'
import json, sys
lc = sys.argv[1]
d = json.loads(open(f"gpurun_out/c_bench_{lc}.log").read().strip().split("\n")[-1])
k = d["kernels"]
print(lc, "ms/V-cycle", round(d["ms_per_step"], 3), "fwd", k["tk_forward_subst"]["ms"], "back", k["tk_sgs_back_half"]["ms"], "coarse its", d.get("coarse_share", {}).get("share"))
PY
done
