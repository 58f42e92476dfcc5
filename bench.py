#!/usr/bin/env python
"""Benchmark of the B200 multigrid-in-time KKT preconditioner.

Metric (BASELINE.json): V-cycle time-step.DoF/s -- per V-cycle application,
the number of time steps times the KKT unknowns per step (4 N_u + N_z),
divided by the application time -- plus the full MG-preconditioned FGMRES
solve time.  One "step" = one V-cycle application of the rediscretised
hierarchy (pre-smooth, residual-restrict, recursion, SGS-GMRES coarse solve,
prolong-correct, post-smooth) to one right-hand side resident in HBM.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl ours|reference]

Prints ONE JSON line (rank 0).  See DESIGN.md for the contract details.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0}


# ncu-measured DRAM traffic per C-ABI call, from the committed capture of the
# SAME configuration (tools/round_profile.sh / tools/cfg4_profile.sh write
# profiles/<NCU_TAG>_cfg<N>_ncu_summary.json): the fine-level launch of the
# `--set full` capture whose kernel matches the call's pattern for the level's
# structure family (TRI: Burgers; DENSE: van der Pol), or the summed launch-list
# entries of the kernels one call launches.
NCU_TAG = "r02"
def _targs(kernel: str):
    """Template arguments of a kernel name ("void f<4, 0, 1>" -> ["4", "0", "1"])."""
    k = kernel.split("(")[0]
    if "<" not in k:
        return []
    return [t.strip() for t in k[k.index("<") + 1:k.rindex(">")].split(",")]


def _t(kernel: str, i: int):
    a = _targs(kernel)
    return a[i] if i < len(a) else "0"


# call -> (TRI predicate, DENSE predicate) on the kernel name;
# tri_rows_part<W, MODE, FULL, CL, RJ, TOE>, dense_rows<NU, NZ, MODE>
_NCU_FULL = {
    "tk_jacobi_sweep": (lambda k: "tri_rows_part<" in k and _t(k, 1) in ("0", "3")
                        and _t(k, 4) == "0" and _t(k, 6) == "0",
                        lambda k: "dense_rows_split<" in k or ("dense_rows<" in k and _t(k, 2) == "4")),
    "tk_jacobi0_restrict": (lambda k: "tri_rows_part<" in k and _t(k, 1) == "3"
                            and _t(k, 4) == "1",
                            lambda k: "dense_rows<" in k and _t(k, 2) == "4"),
    "tk_jacobi0_restrict_um": (lambda k: "tri_rows_part<" in k and _t(k, 1) == "3"
                               and _t(k, 4) == "1",
                               lambda k: "dense_rows_split<" in k),
    "tk_jacobi_prolong": (lambda k: "tri_rows_part<" in k and _t(k, 1) == "3"
                          and _t(k, 6) == "1",
                          lambda k: "dense_rows_split<" in k),
    "tk_residual_restrict": (lambda k: "tri_resrestrict" in k,
                             lambda k: "dense_rows<" in k and _t(k, 2) == "2"),
    "tk_prolong_add": (lambda k: "prolong_rows_kernel" in k, lambda k: "prolong_small_kernel" in k),
    "tk_kkt_apply": (lambda k: "tri_apply<0" in k,
                     lambda k: "dense_rows<" in k and _t(k, 2) == "0"),
    "tk_residual_restrict_jacobi0": (lambda k: "restrict_jacobi0_rows" in k,
                                     lambda k: "restrict_jacobi0_small" in k),
}
_NCU_NAMES = {"tk_jacobi_sweep": ("tri_rows_part<W, 3, ., CL, 0, .>", "dense_rows<NU, NZ, 4>"),
              "tk_jacobi0_restrict": ("tri_rows_part<W, 3, ., CL, 1, .>", "dense_rows<NU, NZ, 4>"),
              "tk_jacobi0_restrict_um": ("tri_rows_part<W, 3, ., CL, 1, ., 0>", "dense_rows_split<NU, NZ>"),
              "tk_jacobi_prolong": ("tri_rows_part<W, 3, ., CL, 0, ., 1>", "dense_rows_split<NU, NZ>"),
              "tk_residual_restrict": ("tri_resrestrict", "dense_rows<NU, NZ, 2>"),
              "tk_prolong_add": ("prolong_rows_kernel", "prolong_small_kernel"),
              "tk_kkt_apply": ("tri_apply<0>", "dense_rows<NU, NZ, 0>"),
              "tk_residual_restrict_jacobi0": ("restrict_jacobi0_rows", "restrict_jacobi0_small")}
_NCU_KERNELS = {
    "tk_forward_subst": ("tri_rows_part<4, 3, 1, 1, 0, 1, 0, 4", "tri_chainw_kernel<1", "tri_chainw_kernel<1",
                         "tri_chain_carry_seg<1", "tri_chain_carry_seg<1", "tri_rows_part<4, 1,"),
    "tk_backward_subst": ("tri_chainw_kernel<0", "tri_chainw_kernel<0", "tri_chain_carry_seg<0",
                          "tri_chain_carry_seg<0", "tri_rows_part<4, 2,"),
    "tk_sgs_back_half": ("tri_chainw_kernel<0", "tri_chainw_kernel<0", "tri_chain_carry_seg<0",
                         "tri_chain_carry_seg<0", "tri_rows_part<4, 4,"),
}


def ncu_traffic(call: str, config: int, family: int):
    """DRAM bytes per call from the committed ncu summary of this config, or
    (None, source) when no capture of a matching kernel exists."""
    src = f"{NCU_TAG}_cfg{config}_ncu_summary.json"
    path = os.path.join(ROOT, "profiles", src)
    if not os.path.exists(path):
        return None, None
    with open(path) as fh:
        summ = json.load(fh)
    if call in _NCU_FULL:
        pred = _NCU_FULL[call][0 if family == 1 else 1]
        fine = [d for d in summ["full_capture"] if pred(d["kernel"])]
        if fine:
            # the u/mu-only pre-smoothing shares its kernel name with the full one (the
            # partial store is a runtime flag): it is the capture that wrote fewer bytes
            pick = min if call == "tk_jacobi0_restrict_um" else max
            d = pick(fine, key=lambda e: e["dram_write_MB"] if call.startswith("tk_jacobi0_restrict")
                     else e["duration_us"])
            return int((d["dram_read_MB"] + d["dram_write_MB"]) * 1e6), src
        return None, src
    pats = _NCU_KERNELS.get(call) if family == 1 else None
    if not pats:
        return None, src
    tot = 0
    for pat in pats:
        for d in summ["launch_list"]:
            if pat in d["kernel"]:
                tot += d["dram_bytes_per_launch"]
                break
    return (tot or None), src


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return d, "measured"
    except Exception:
        return PEAKS_FALLBACK, "fallback"


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.lines = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.index)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"],
                    "samples": 0}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, val in zip(names, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------ CPU reference
def oracle_sample(index: int):
    """Bounded sample of configs[index] for the CPU reference (the oracle
    restatement of tempokkt, dense per-block inverses as the reference)."""
    from oracle import tk_oracle as O
    from paper_2405_04808_b200 import configs
    p = dict(configs.CONFIGS[index])
    if p["problem"] == "vanderpol":
        nt, levels = 4096, min(p["levels"], 8)
        prob = O.vanderpol(mu=p["mu"], alpha=p["alpha"], n_controls=p["n_controls"],
                           u0=p["u0"], theta=p["theta"])
        nz = p["n_controls"]
        xs = None
    else:
        nt, levels = 8, 3
        prob = O.burgers(n_u=p["nx"], nu=p["nu"], alpha=p["alpha"], theta=p["theta"],
                         u0_kind=p["u0_kind"])
        nz = p["nx"]
        xs = np.arange(1, p["nx"] + 1) / (p["nx"] + 1.0)
    from paper_2405_04808_b200.timedisc import TimeGrid
    dt_full = p["t_final"] / p["nt"]
    grid = TimeGrid(dt_full * nt, nt)       # same dt as the full workload, fewer steps
    pp = dict(p, nt=nt, t_final=grid.t_final)
    z = configs._controls(pp, grid, nz, xs)
    states = O.forward_solve(prob, z, nt, grid.dt)
    h = O.build_hierarchy(prob, states, states, z, nt, grid.dt, levels, sweeps=1,
                          cycle_kind="v", coarse_tol=1e-2)
    b = np.random.default_rng(p["seed"]).standard_normal(h.levels[0].kkt.dim)
    desc = f"configs[{index}] shape at nt={nt} (same dt, n_u, n_z), {levels}-level V(1,1)"
    return h, b, nt * (4 * prob.n_u + prob.n_z), desc


def cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        n = max((d.get("num_threads") or 1) for d in threadpool_info())
        return int(n)
    except Exception:
        return os.cpu_count() or 1


def time_oracle(index: int, steps: int, warmup: int, budget_s: float = 20.0):
    from oracle import tk_oracle as O
    h, b, unknowns, desc = oracle_sample(index)
    for _ in range(warmup):
        O.cycle(h, 0, b)
    t0 = time.perf_counter()
    done = 0
    while done < steps:
        O.cycle(h, 0, b)
        done += 1
        if time.perf_counter() - t0 > budget_s and done >= 1:
            break
    dt = (time.perf_counter() - t0) / done
    return unknowns / dt, desc + f", {done} timed V-cycles", done


# ------------------------------------------------------------------ ours
def solve_once(P, h, b, setup):
    """One full MG-FGMRES solve (krylov.py:204-210 around multigrid.py:304-311),
    wall time with a device synchronisation on both sides."""
    import torch
    S = setup.solver
    torch.cuda.empty_cache()                      # cached blocks back to the driver
    free, _ = torch.cuda.mem_get_info()
    per_it = 2 * setup.dim * 8                    # V and Z columns
    m_fit = int(0.9 * free // per_it) - 4         # (+ x, r, w and V-cycle temporaries)
    restart = None if m_fit >= S["max_iters"] + 1 else max(2, m_fit)
    h.stats = type(h.stats)()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, rep = P.fgmres(h.levels[0].kkt.as_operator(), P.mg_preconditioner(h), b,
                      rel_tol=S["rel_tol"], max_iters=S["max_iters"], restart=restart)
    torch.cuda.synchronize()
    secs = time.perf_counter() - t0
    del x
    return {"config": f"configs[{setup.index}] {setup.describe()}", "seconds": round(secs, 4),
            "outer": "fgmres", "restart": restart, "iterations": rep.iterations,
            "final_rel_residual": rep.final_relative_residual,
            "coarse_iters_avg": h.stats.average,
            "note": ("rel_tol 1e-8 is not reached within 401 iterations: the reference does the "
                     "same (q_z = dt*w_control, timedisc.py:194-206; configs[1] at full size "
                     "matches the reference's own run, tests/golden/cfg1_full_solve.npz)")
            if rep.final_relative_residual > S["rel_tol"] else ""}


def run_ours(args, rank, world, local_rank):
    import torch
    torch.cuda.set_device(local_rank)
    import paper_2405_04808_b200 as P
    from paper_2405_04808_b200 import configs, device as dev, roofline
    from paper_2405_04808_b200.krylov import vec_ops

    if world > 1:
        from paper_2405_04808_b200 import slabs
        return slabs.bench_rank(args, rank, world, local_rank)

    setup = configs.build_setup(args.config)
    S = setup.solver
    h = P.build_hierarchy(setup.problem, setup.u, setup.v, setup.z, setup.grid, setup.levels,
                          sweeps=S["sweeps"], omega=S["omega"], cycle_kind=S["cycle"],
                          coarse_tol=S["coarse_tol"], coarse_max_iters=S["coarse_max_iters"])
    r_host = setup.rhs()
    r_dev = dev.to_device(r_host)
    prec = P.mg_preconditioner(h)
    stream = torch.cuda.current_stream()
    unknowns = setup.grid.n_steps * setup.dof_per_step

    for _ in range(max(args.warmup, 1)):
        prec(r_dev)
    torch.cuda.synchronize()

    # per-kernel breakdown from one untimed profiled step (events around every call)
    names = {"tk_jacobi_sweep", "tk_residual_restrict", "tk_prolong_add", "tk_forward_subst",
             "tk_backward_subst", "tk_sgs_back_half", "tk_kkt_apply", "tk_kkt_apply_diag",
             "tk_kkt_residual", "tk_dot", "tk_nrm2", "tk_axpy", "tk_scale_into", "tk_rsub",
             "tk_gemv_t_add", "tk_arnoldi_mgs", "tk_copy_kernel", "tk_residual_restrict_jacobi0",
             "tk_jacobi0_restrict", "tk_jacobi0_restrict_um", "tk_jacobi_prolong"}
    # (eager cycles: the CUDA-graph replay hides the coarse levels' kernels)
    from paper_2405_04808_b200 import graph as G
    graph_on = G.ENABLED
    G.ENABLED = False
    eager_steps = 3
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ea.record(stream)
    for _ in range(eager_steps):
        prec(r_dev)
    eb.record(stream)
    torch.cuda.synchronize()
    eager_ms = ea.elapsed_time(eb) / eager_steps
    dev.INSTR.timed, dev.INSTR.records = names, []
    prec(r_dev)
    torch.cuda.synchronize()
    G.ENABLED = graph_on
    per = {}
    for nm, a, e0, e1 in dev.INSTR.records:
        ms = e0.elapsed_time(e1)
        d = per.setdefault(nm, {"calls": 0, "ms": 0.0, "bytes": 0})
        d["calls"] += 1
        d["ms"] += ms
        d["bytes"] += roofline.algorithmic_bytes(nm, a)
    fine_recs = {}
    for nm, a, e0, e1 in dev.INSTR.records:   # fine-level launch of each HBM kernel
        if nm in ("tk_jacobi_sweep", "tk_residual_restrict", "tk_residual_restrict_jacobi0",
                  "tk_jacobi0_restrict", "tk_jacobi0_restrict_um", "tk_jacobi_prolong"):
            lvl = roofline.dim_of(a[0]._obj)
        elif nm == "tk_prolong_add":
            lvl = int(a[0]) * (4 * int(a[1]) + int(a[2]))
        else:
            continue
        cur = fine_recs.get(nm)
        if cur is None or lvl > cur[0]:
            fine_recs[nm] = (lvl, [(a, e0.elapsed_time(e1))])
        elif lvl == cur[0]:
            cur[1].append((a, e0.elapsed_time(e1)))
    # coarse-solve share of the (eager) V-cycle: every call on the coarsest
    # level (SGS substitutions, operator, Krylov vector kernels of its GMRES)
    nc_dim = h.levels[-1].kkt.dim
    coarse_ms = 0.0
    for nm, a, e0_, e1_ in dev.INSTR.records:
        lv = getattr(a[0], "_obj", None) if a else None
        on_coarse = (roofline.dim_of(lv) == nc_dim) if lv is not None else \
            (isinstance(a[0], int) and int(a[0]) == nc_dim)
        if on_coarse:
            coarse_ms += e0_.elapsed_time(e1_)
    tot_ms = sum(v["ms"] for v in per.values())
    coarse_share = {"share": coarse_ms / tot_ms if tot_ms else None, "coarse_ms": coarse_ms,
                    "cycle_kernels_ms": tot_ms, "coarse_steps": h.levels[-1].n_steps,
                    "how": "CUDA events around every C-ABI call of one eager V-cycle; calls "
                           "on the coarsest level (SGS-GMRES: substitutions, operator, "
                           "Krylov vector kernels) over all calls"}
    dev.INSTR.timed, dev.INSTR.records = None, []
    dominant_eager = max(per, key=lambda k: per[k]["ms"])
    # the fine-level KKT mat-vec (the outer Krylov operator), timed on its own
    a0 = h.levels[0].kkt
    y0 = dev.empty(a0.dim)
    dev.INSTR.timed, dev.INSTR.records = {"tk_kkt_apply"}, []
    for _ in range(5):
        dev.call("tk_kkt_apply", a0.lref, dev.P(r_dev), dev.P(y0), dev.stream())
    torch.cuda.synchronize()
    fine_recs["tk_kkt_apply"] = (a0.dim, [(a, s_.elapsed_time(t_)) for _, a, s_, t_ in dev.INSTR.records[1:]])
    dev.INSTR.timed, dev.INSTR.records = None, []

    # timed region: K V-cycles, CUDA events on the launching stream; the
    # dominant kernel's launches are bracketed by events for the roofline
    clk = ClockSampler(local_rank)
    clk.start()
    time.sleep(0.3)
    dev.INSTR.timed, dev.INSTR.records = set(names), []
    dev.INSTR.counting, dev.INSTR.launches = True, 0
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        prec(r_dev)
    e1.record(stream)
    torch.cuda.synchronize()
    total_ms = e0.elapsed_time(e1)
    launches = dev.INSTR.launches
    recs = dev.INSTR.records
    dev.INSTR.timed, dev.INSTR.records, dev.INSTR.counting = None, [], False
    clocks = clk.stop()
    ms_step = total_ms / args.steps
    value = unknowns / (ms_step * 1e-3)

    def kernel_stats(nm, fine_only=False):
        rs = [(a, s.elapsed_time(t)) for n_, a, s, t in recs if n_ == nm]
        if not rs:
            return 0.0, float("nan"), 0
        if fine_only:
            top = max(roofline.dim_of(a[0]._obj) for a, _ in rs)
            rs = [(a, ms) for a, ms in rs if roofline.dim_of(a[0]._obj) == top]
        byts = sum(roofline.algorithmic_bytes(nm, a) for a, _ in rs)
        ms = sum(m for _, m in rs)
        return byts / len(rs), ms / len(rs), len(rs)

    peaks, peak_kind = load_peaks()
    hbm = float(peaks["hbm_gbs"])
    fam = int(h.levels[0].kkt.family)
    hbm_kernels = {}
    for nm, (_, rs) in fine_recs.items():
        byts = sum(roofline.algorithmic_bytes(nm, a) for a, _ in rs) / len(rs)
        ms = sum(m for _, m in rs) / len(rs)
        achk = byts / (ms * 1e-3) / 1e9
        tr, tsrc = ncu_traffic(nm, args.config, fam)
        hbm_kernels[nm] = {"level": "fine", "bytes_per_launch": byts, "ms_per_launch": ms,
                           "achieved_GBps": achk, "frac": achk / hbm,
                           "ncu_kernel": _NCU_NAMES[nm][0 if fam == 1 else 1]
                           if nm in _NCU_NAMES else None,
                           "traffic": tr, "traffic_source": tsrc}
    # dominant kernel = the C-ABI call with the most device time among those
    # launched in the timed region (the graphed coarse levels replay as one
    # launch; their share is reported in `coarse_share`)
    tot_by = {}
    for n_, a, s_, t_ in recs:
        tot_by[n_] = tot_by.get(n_, 0.0) + s_.elapsed_time(t_)
    dominant = max(tot_by, key=tot_by.get)
    b_dom, ms_dom, n_dom = kernel_stats(dominant)
    ach = b_dom / (ms_dom * 1e-3) / 1e9
    # the fine-level post-smoothing sweep (with the prolongation inside on V(1,1) levels)
    jac_name = "tk_jacobi_prolong" if any(n_ == "tk_jacobi_prolong" for n_, *_ in recs) \
        else "tk_jacobi_sweep"
    b_j, ms_j, n_j = kernel_stats(jac_name, fine_only=True)
    ach_j = b_j / (ms_j * 1e-3) / 1e9

    # e2e through the public API with pinned host buffers: every step copies its
    # rhs in and its result out.  Serial: prec(r) between blocking copies;
    # pipelined (HostPipeline): copy-in k+1 / V-cycle k / copy-out k-1 overlap.
    r_pin = torch.from_numpy(r_host).pin_memory()
    out_pins = [torch.empty(r_host.shape[0], dtype=torch.float64).pin_memory() for _ in range(2)]
    e2e_steps = max(2, min(args.steps, 5))
    for _ in range(1):
        r_dev.copy_(r_pin, non_blocking=True)
        out_pins[0].copy_(prec(r_dev), non_blocking=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(e2e_steps):
        r_dev.copy_(r_pin, non_blocking=True)
        out_pins[0].copy_(prec(r_dev), non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_serial_ms = e0.elapsed_time(e1) / e2e_steps
    pipe = P.HostPipeline(prec, setup.dim)
    pipe_steps = max(4, args.steps)
    ins = [r_pin] * pipe_steps
    outs = [out_pins[k & 1] for k in range(pipe_steps)]
    pipe.run(ins[:2], outs[:2])
    torch.cuda.synchronize()
    e0.record(stream)
    pipe.run(ins, outs, start_event=e0)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / pipe_steps

    # full MG-FGMRES solves (tol 1e-8, <= 401 its): the benched configuration
    # itself, on the same hierarchy and rhs (restart sized to the free HBM,
    # since V and Z hold 2 vectors per iteration), and configs[1], whose
    # full-size solve is pinned to the reference's own run
    solves = {}
    for sc in ([args.config] + [c for c in args.solve_configs if c != args.config]
               if args.solve_config >= 0 else []):
        if sc == args.config:
            hs, bs, ss = h, r_dev, setup
        else:
            ss = configs.build_setup(sc)
            S2 = ss.solver
            hs = P.build_hierarchy(ss.problem, ss.u, ss.v, ss.z, ss.grid, ss.levels,
                                   sweeps=S2["sweeps"], cycle_kind=S2["cycle"],
                                   coarse_tol=S2["coarse_tol"])
            bs = dev.to_device(ss.rhs())
        solves[sc] = solve_once(P, hs, bs, ss)
        if sc != args.config:
            del hs, bs
            torch.cuda.empty_cache()
    solve = solves.get(args.config)
    solve_cfg1 = solves.get(1) if args.config != 1 else None

    cpu = None
    if not args.no_cpu_baseline:
        v_cpu, desc, n_cpu = time_oracle(args.config, steps=3, warmup=1)
        cpu = {"value": v_cpu, "unit": "time-step*DoF/s", "cores": cpu_threads(),
               "kind": "port", "sample": desc}

    line = {
        "metric": "V-cycle time-step*DoF/s (fp64) + full MG-FGMRES solve time",
        "value": value, "unit": "time-step*DoF/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: forward-march linearisation + N(0,1) rhs (seeded)",
        "config": {"workload": f"configs[{args.config}] {setup.describe()}",
                   "n_steps": setup.grid.n_steps, "n_u": setup.n_u, "n_z": setup.n_z,
                   "levels": setup.levels, "cycle": "V(1,1) block-Jacobi, coarse SGS-GMRES 1e-2",
                   "kkt_dim": setup.dim, "parallelism": f"time-slabs x{world}",
                   "l2": "inputs larger than L2" if setup.dim * 8 > 126e6 else
                         "inputs smaller than L2 (no flush)"},
        "e2e": {"value": unknowns / (e2e_ms * 1e-3), "unit": "time-step*DoF/s",
                "h2d_bytes_per_step": int(r_host.nbytes), "d2h_bytes_per_step": int(r_host.nbytes),
                "ms_per_step": e2e_ms, "steps": pipe_steps,
                "api": "HostPipeline(mg_preconditioner(h)).run(pinned rhs -> pinned results): "
                       "copy-in k+1 / V-cycle k / copy-out k-1 on three streams",
                "serial": {"value": unknowns / (e2e_serial_ms * 1e-3), "ms_per_step": e2e_serial_ms,
                           "api": "mg_preconditioner(h)(r) between blocking pinned copies"}},
        "roofline": {"bound": "hbm", "kernel": dominant, "achieved": ach,
                     "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                     "traffic": ncu_traffic(dominant, args.config, fam)[0],
                     "traffic_source": ncu_traffic(dominant, args.config, fam)[1],
                     "peak_kind": peak_kind, "launches_timed": n_dom,
                     "bytes_per_launch": b_dom, "ms_per_launch": ms_dom,
                     "note": ("the Gauss-Seidel substitutions are serial in time (one CTA walks "
                              "the coarse intervals): latency-bound, not HBM-bound"
                              if "subst" in dominant else ""),
                     "fine_jacobi": {"call": jac_name, "achieved": ach_j, "frac": ach_j / hbm,
                                     "bytes_per_launch": b_j, "ms_per_launch": ms_j,
                                     "traffic": ncu_traffic(jac_name, args.config,
                                                            fam)[0]}},
        "hbm_kernels": hbm_kernels,
        "kernels": {k: {"calls": v["calls"], "ms": round(v["ms"], 4),
                        "share": round(v["ms"] / sum(x["ms"] for x in per.values()), 4),
                        "GBps": round(v["bytes"] / (v["ms"] * 1e-3) / 1e9, 1) if v["ms"] else None}
                    for k, v in sorted(per.items(), key=lambda kv: -kv[1]["ms"])},
        "gpu_launches": launches,
        "vcycle_graph": {"enabled": graph_on,
                         "api": "levels 1..L-1 incl. the coarse SGS-GMRES (device WHILE loop) "
                                "replayed as one CUDA graph per V-cycle",
                         "eager_ms_per_step": eager_ms},
        "clocks": clocks,
        "cpu_baseline": cpu,
        "solve": solve,
        "solve_cfg1": solve_cfg1,
        "coarse_share": coarse_share,
    }
    return line


def run_reference(args, rank, world):
    if rank != 0:
        return None
    v, desc, n = time_oracle(args.config, steps=max(args.steps, 1), warmup=args.warmup,
                             budget_s=60.0)
    cores = cpu_threads()
    return {"impl": "reference",
            "metric": "V-cycle time-step*DoF/s (fp64) + full MG-FGMRES solve time",
            "value": v, "unit": "time-step*DoF/s", "n_gpus": world, "steps": n,
            "warmup": args.warmup, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"configs[{args.config}] (bounded CPU sample)"},
            "cpu_baseline": {"value": v, "unit": "time-step*DoF/s", "cores": cores,
                             "kind": "port", "sample": desc},
            "e2e": {"value": v, "unit": "time-step*DoF/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--solve-config", type=int, default=0,
                    help="-1: no full solves (default: the benched config + configs[1])")
    ap.add_argument("--solve-configs", type=lambda t: [int(c) for c in t.split(",") if c],
                    default=[1])
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        line = run_reference(args, rank, world)
    else:
        line = run_ours(args, rank, world, local_rank)
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
