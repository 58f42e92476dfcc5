#!/bin/bash
# Jacobi kernel change: size-sweep + parity GPU tests, fine-sweep timing, short bench
timeout 900 python -m pytest tests/test_gpu_sizes.py tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_slabs_gpu.py -x -q > gpurun_out/j_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/j_tests.log
timeout 300 python tools/time_jacobi.py 2 new 2>&1 | tail -1
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --solve-config -1 > gpurun_out/j_bench.json 2> gpurun_out/j_bench.err; echo "bench rc=$?"
python3 - <<'PY'
import json
d = json.loads(open("gpurun_out/j_bench.json").read().strip().split("\n")[-1])
print("ms/V-cycle", round(d["ms_per_step"], 3), "value", "%.3e" % d["value"])
fj = d["roofline"]["fine_jacobi"]
print("fine jacobi ms", round(fj["ms_per_launch"], 4), "frac", round(fj["frac"], 3))
print({k: v["ms"] for k, v in d["kernels"].items()})
PY
