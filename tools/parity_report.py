"""Print measured GPU-vs-reference discrepancies for every golden case
(diagnostic companion of tests/test_gpu_parity.py).  Run on a B200."""

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from conftest import CASES, load_golden, product_problem, rel  # noqa: E402

import paper_2405_04808_b200 as P  # noqa: E402


def main(cases):
    for name in cases:
        g = load_golden(name)
        p, grid = product_problem(g)
        t0 = time.time()
        st = P.build_stage_blocks(p, grid.dt, g["u"], g["v"], g["z"])
        a = P.assemble_kkt(st)
        out = {}
        out["Ax"] = rel(a.apply(g["x"]), g["Ax"])
        out["Dinv"] = rel(P.DiagonalSolver(a).solve_all(g["b"]), g["Dinv_b"])
        out["jac2"] = rel(P.jacobi_apply(a, None, g["b"], g["x"], 2), g["jac2"])
        out["fgs"] = rel(P.fgs_apply(a, None, g["b"], g["x"]), g["fgs"])
        out["bgs"] = rel(P.bgs_apply(a, None, g["b"], g["x"]), g["bgs"])
        out["sgs"] = rel(P.sgs_apply(a, None, g["b"], g["x"]), g["sgs"])
        h = P.build_hierarchy(p, g["u"], g["v"], g["z"], grid, int(g["levels"]),
                              sweeps=int(g["sweeps"]), coarse_tol=1e-2)
        t = h.transfers[0]
        out["restrict_exact"] = bool(np.array_equal(t.restrict_kkt(g["x"]), g["restrict_x"]))
        out["prolong_exact"] = bool(np.array_equal(t.prolong_kkt(g["xc"]), g["prolong_xc"]))
        xc = P.coarse_solve(h, g["coarse_r"])
        out["coarse"] = (rel(xc, g["coarse_x"]), h.stats.iters, int(g["coarse_iters"]))
        for kind in ("v", "w", "f"):
            h.cycle_kind = kind
            h.stats = type(h.stats)()
            c = P.cycle(h, 0, g["b"])
            out[f"cycle_{kind}"] = (rel(c, g[f"cycle_{kind}"]), h.stats.iters,
                                    int(g[f"cycle_{kind}_coarse_iters"]))
        h.cycle_kind = "v"
        for outer in ("fgmres", "gmres"):
            h.stats = type(h.stats)()
            fn = P.fgmres if outer == "fgmres" else P.gmres
            ts = time.time()
            x, rep = fn(a.as_operator(), P.mg_preconditioner(h), g["b"], rel_tol=1e-8,
                        max_iters=401)
            out[outer] = dict(x=rel(x, g[f"{outer}_x"]),
                              hist=rel(np.array(rep.residual_history), g[f"{outer}_hist"])
                              if len(rep.residual_history) == len(g[f"{outer}_hist"]) else "len",
                              iters=(rep.iterations, int(g[f"{outer}_iters"])),
                              coarse=(h.stats.iters, int(g[f"{outer}_coarse_iters"])),
                              secs=round(time.time() - ts, 2))
        print(f"== {name} ({time.time() - t0:.1f}s)")
        for k, v in out.items():
            print(f"   {k:16s} {v}")
        sys.stdout.flush()


if __name__ == "__main__":
    main(sys.argv[1:] or CASES)
