#!/bin/bash
# GPU tests for the TRI sizes + a short bench; prints the fine-Jacobi roofline and the per-call breakdown
timeout 600 python -m pytest tests/test_gpu_sizes.py tests/test_gpu_parity.py -x -q > gpurun_out/t_sizes.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/t_sizes.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --solve-config -1 > gpurun_out/bench2.log 2>&1
echo "bench rc=$?"
python3 - <<'PY'
import json
d = json.loads(open("gpurun_out/bench2.log").read().strip().split("\n")[-1])
print("ms/V-cycle", round(d["ms_per_step"], 3), "value", "%.3e" % d["value"])
fj = d["roofline"]["fine_jacobi"]
print("fine jacobi ms", round(fj["ms_per_launch"], 4), "frac", round(fj["frac"], 3))
print({k: v["ms"] for k, v in d["kernels"].items()})
PY
