#!/bin/bash
# configs[4] (Burgers nx=2048, nt=65536, 8 levels) evidence on one B200:
# bench line, ncu launch list of one V-cycle (per-kernel share incl. the coarse
# solve), one --set full capture of each fine-level n_u=2048 HBM kernel.
# usage: tools/cfg4_profile.sh <tag>   (summaries in gpurun_out/, the .ncu-rep in /tmp)
tag=${1:-r02}
timeout 900 python bench.py --config 4 --steps 5 --warmup 3 --solve-config -1 --no-cpu-baseline > gpurun_out/${tag}_bench_cfg4.json 2> gpurun_out/${tag}_bench_cfg4.err; echo "bench cfg4 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  python tools/prof_vcycle.py 4 1 > gpurun_out/${tag}_cfg4_launches.csv 2> gpurun_out/${tag}_cfg4_launches.err; echo "ncu cfg4 list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"tri_apply|tri_rows_part|tri_resrestrict|prolong_rows|restrict_jacobi0|tri_rows_rec" -s 1 -c 8 \
  -o /tmp/${tag}_cfg4_full python tools/prof_kernels.py 4 > gpurun_out/${tag}_cfg4_full.log 2>&1; echo "ncu cfg4 full rc=$?"
python tools/ncu_summary.py gpurun_out/${tag}_cfg4_launches.csv /tmp/${tag}_cfg4_full.ncu-rep gpurun_out/${tag}_cfg4_ncu > /dev/null 2>&1; echo "summary rc=$?"
ncu -i /tmp/${tag}_cfg4_full.ncu-rep --page raw --csv > gpurun_out/${tag}_cfg4_full_raw.csv 2>/dev/null; echo "raw rc=$?"
ls -la /tmp/${tag}_cfg4_full.ncu-rep
