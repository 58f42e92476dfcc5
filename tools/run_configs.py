"""Time one V-cycle (and optionally the full MG-FGMRES solve) for each
BASELINE configuration on the GPU.  Usage: python tools/run_configs.py 0 1 3 [--solve]"""

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2405_04808_b200 as P  # noqa: E402
from paper_2405_04808_b200 import configs, device as dev  # noqa: E402


def main():
    idxs = [int(a) for a in sys.argv[1:] if a.isdigit()]
    solve = "--solve" in sys.argv
    for i in idxs:
        t0 = time.perf_counter()
        s = configs.build_setup(i)
        t_setup = time.perf_counter() - t0
        S = s.solver
        t0 = time.perf_counter()
        h = P.build_hierarchy(s.problem, s.u, s.v, s.z, s.grid, s.levels, sweeps=S["sweeps"],
                              cycle_kind=S["cycle"], coarse_tol=S["coarse_tol"])
        torch.cuda.synchronize()
        t_h = time.perf_counter() - t0
        r = dev.to_device(s.rhs())
        prec = P.mg_preconditioner(h)
        for _ in range(2):
            prec(r)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h.stats = type(h.stats)()
        e0.record()
        k = 5
        for _ in range(k):
            prec(r)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / k
        out = dict(config=i, name=s.describe(), dim=s.dim, setup_s=round(t_setup, 2),
                   hierarchy_s=round(t_h, 2), vcycle_ms=round(ms, 3),
                   coarse_its_per_cycle=h.stats.iters / k,
                   tsdof_per_s=s.grid.n_steps * s.dof_per_step / (ms * 1e-3))
        print(json.dumps(out), flush=True)
        if solve:
            # (F)GMRES keeps V and Z: size the restart to the free HBM
            free, _ = torch.cuda.mem_get_info()
            free += torch.cuda.memory_reserved() - torch.cuda.memory_allocated()
            per_it = 2 * s.dim * 8
            m_fit = int(0.85 * free // per_it) - 2
            restart = None if m_fit >= S["max_iters"] + 1 else max(2, m_fit)
            out = dict(config=i, name=s.describe(), restart=restart)
            h.stats = type(h.stats)()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            x, rep = P.fgmres(h.levels[0].kkt.as_operator(), prec, r, rel_tol=S["rel_tol"],
                              max_iters=S["max_iters"], restart=restart)
            torch.cuda.synchronize()
            out.update(solve_s=round(time.perf_counter() - t0, 3), iters=rep.iterations,
                       final_rel=rep.final_relative_residual,
                       coarse_its_avg=h.stats.average)
            print(json.dumps(out), flush=True)
            del x
        del h, r, prec
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
