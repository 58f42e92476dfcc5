"""Summarise ncu outputs into profiles/: the per-launch list (gpu__time_duration
+ dram bytes, cold-cache and serialised) and one `--set full` capture.

usage: python tools/ncu_summary.py <launches.csv> <full.ncu-rep> <out_prefix>
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict


def launches(path):
    txt = open(path).read()
    start = txt.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[start:])))
    per = defaultdict(lambda: defaultdict(float))
    for r in rows:
        k = r["Kernel Name"].split("(")[0]
        m = r["Metric Name"]
        try:
            v = float(r["Metric Value"].replace(",", ""))
        except ValueError:
            continue
        unit = r.get("Metric Unit", "")
        if m == "gpu__time_duration.sum":
            per[k]["ns"] += v * {"us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6,
                                 "s": 1e9, "second": 1e9}.get(unit, 1.0)
            per[k]["n"] += 1
        elif m.startswith("dram__bytes"):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
                     "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)
            per[k]["bytes"] += v * scale
    # one-off hierarchy setup (stage linearisation, factor records, chunk and
    # group propagators) is listed but excluded from the V-cycle shares
    setup = ("tri_chain_kernel<1, 0, 1,", "tri_factor_kernel", "stage_", "tri_transpose",
             "check_k_kernel", "check_blocks_kernel", "FillFunctor", "tri_chainw_factor")
    is_setup = {k: any(s in k for s in setup) for k in per}
    tot = sum(d["ns"] for k, d in per.items() if not is_setup[k])
    out = []
    for k, d in sorted(per.items(), key=lambda kv: (is_setup[kv[0]], -kv[1]["ns"])):
        out.append(dict(kernel=k, setup=is_setup[k], launches=int(d["n"]),
                        total_us=round(d["ns"] / 1e3, 1),
                        share=None if is_setup[k] else round(d["ns"] / tot, 4),
                        dram_bytes_per_launch=int(d["bytes"] / max(d["n"], 1)),
                        dram_GBps=round(d["bytes"] / max(d["ns"], 1), 1)))
    return out


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    units = dict(zip(hdr, rows[1]))
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v)
                  for k, v in d.items()
                  if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith(
                      "not_issued") and v not in ("", "n/a") and float(v) > 0}
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:4]
        tot = sum(stalls.values()) or 1.0

        def f(key):
            try:
                v = float(d.get(key, "nan").replace(",", ""))
            except ValueError:
                return float("nan")
            u = units.get(key, "")
            scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3,
                     "B": 1e-6, "KB": 1e-3, "MB": 1.0, "GB": 1e3,
                     "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6,
                     "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}.get(u, 1.0)
            return v * scale
        dur_us = f("gpu__time_duration.sum")
        rd, wr = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")
        res.append(dict(kernel=d["Kernel Name"].split("(")[0], grid=d.get("Grid Size"),
                        block=d.get("Block Size"), duration_us=dur_us,
                        dram_read_MB=rd, dram_write_MB=wr,
                        dram_GBps=round((rd + wr) / dur_us * 1e3, 1) if dur_us else None,
                        dram_pct_peak=f("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                        regs=f("launch__registers_per_thread"),
                        warps_active_pct=f("sm__warps_active.avg.pct_of_peak_sustained_active"),
                        stalls=[(k, round(v / tot, 3)) for k, v in top]))
    return res


if __name__ == "__main__":
    lpath, fpath, prefix = sys.argv[1:4]
    L = launches(lpath)
    F = full(fpath)
    with open(prefix + "_summary.json", "w") as fh:
        json.dump({"launch_list": L, "full_capture": F}, fh, indent=1)
    with open(prefix + "_summary.txt", "w") as fh:
        fh.write("# per-kernel totals from the ncu launch list of one V-cycle after the hierarchy\n"
                 "# build (cold-cache, serialised); setup kernels listed last, share = of the V-cycle\n")
        for d in L:
            fh.write(json.dumps(d) + "\n")
        fh.write("\n# ncu --set full capture\n")
        for d in F:
            fh.write(json.dumps(d) + "\n")
    print(open(prefix + "_summary.txt").read())
