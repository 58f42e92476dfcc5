#!/bin/bash
# graph V-cycle: GPU tests + smoke + short bench (outputs in gpurun_out/)
timeout 600 python -m pytest tests/test_gpu_graph.py -x -q > gpurun_out/g_tests.log 2>&1; echo "graph tests rc=$?"; tail -30 gpurun_out/g_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g_smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/g_smoke.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --solve-config 1 > gpurun_out/g_bench.json 2> gpurun_out/g_bench.err; echo "bench rc=$?"; tail -5 gpurun_out/g_bench.err
python3 - <<'PY'
import json
d = json.loads(open("gpurun_out/g_bench.json").read().strip().split("\n")[-1])
print("ms/V-cycle", round(d["ms_per_step"], 3), "eager", round(d["vcycle_graph"]["eager_ms_per_step"], 3), "value", "%.3e" % d["value"], "e2e ms", round(d["e2e"]["ms_per_step"],3), "launches", d["gpu_launches"])
print("solve", d["solve"])
PY
