#!/bin/bash
# Round-end evidence on one B200: GPU tests, smoke, bench (+ reference arm),
# the ncu launch list of a V-cycle and one --set full capture of each fine-level
# HBM kernel.  usage: tools/round_profile.sh <tag>   (outputs in gpurun_out/)
tag=${1:-r1}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/${tag}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc=$?"
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${tag}_bench_reference.json 2> gpurun_out/${tag}_bench_ref.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  python tools/prof_vcycle.py 2 1 > gpurun_out/${tag}_launches.csv 2> gpurun_out/${tag}_launches.err; echo "ncu list rc=$?"
PROF_GRAPH=1 timeout 600 ncu --profile-from-start off --graph-profiling graph --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  python tools/prof_vcycle.py 2 1 > gpurun_out/${tag}_launches_graph.csv 2> gpurun_out/${tag}_launches_graph.err; echo "ncu graph list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tri_apply|tri_rows_part|tri_resrestrict|prolong_rows|restrict_jacobi0" -s 1 -c 8 \
  -o /tmp/${tag}_full python tools/prof_kernels.py 2 > gpurun_out/${tag}_full.log 2>&1; echo "ncu full rc=$?"
python tools/ncu_summary.py gpurun_out/${tag}_launches.csv /tmp/${tag}_full.ncu-rep gpurun_out/${tag}_ncu > /dev/null 2>&1; echo "summary rc=$?"
python tools/ncu_summary.py gpurun_out/${tag}_launches_graph.csv /tmp/${tag}_full.ncu-rep gpurun_out/${tag}_ncu_graph > /dev/null 2>&1; echo "graph summary rc=$?"
timeout 600 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline --solve-config -1 > gpurun_out/${tag}_bench_cfg3.json 2> gpurun_out/${tag}_bench_cfg3.err; echo "bench cfg3 rc=$?"
timeout 900 python tools/run_configs.py 0 1 3 4 --solve > gpurun_out/${tag}_configs.jsonl 2> gpurun_out/${tag}_configs.err; echo "configs rc=$?"
ncu -i /tmp/${tag}_full.ncu-rep --page raw --csv > gpurun_out/${tag}_full_raw.csv 2>/dev/null; echo "raw rc=$?"
