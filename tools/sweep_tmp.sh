for v in 0 1; do
  if [ $v = 1 ]; then export TK_NO_RECORDS=1; fi
  ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"tri_rows|tri_chain|apply" python tools/prof_vcycle.py 2 1 > gpurun_out/ncu_nr$v.csv 2>/dev/null
  python - $v <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open(f"gpurun_out/ncu_nr{sys.argv[1]}.csv")) if len(r) > 10]
hdr = rows[0]; ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value"); gi = hdr.index("Grid Size")
agg = collections.OrderedDict()
for r in rows[1:]:
    if "<1, 0, 1," in r[ki]: continue
    k = r[ki].split("(")[0][:34] + " " + r[gi]
    a = agg.setdefault(k, [0, 0.0]); a[0] += 1; a[1] += float(r[vi].replace(",", ""))
print("norec", sys.argv[1], {k: (v[0], round(v[1] / v[0] / 1e3, 1)) for k, v in agg.items() if v[1] / v[0] < 200e3})
PY
done
TK_NO_RECORDS=1 python tools/vcycle_time.py 2 norec
python tools/vcycle_time.py 2 rec
