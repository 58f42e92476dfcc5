"""Golden record of the FULL-size BASELINE configs[1] solve, by the REAL reference.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_cfg1_full.py

Burgers nx=128 (interior nodes), nu=0.01, T=1, nt=1024, backward Euler,
sin-step u0, linearised about the forward march under z=0, rhs N(0,1) from
seed 1, 4-level V(1,1) block-Jacobi, coarse SGS-GMRES tol 1e-2, outer
FGMRES tol 1e-8, <= 401 iterations -- the same setup as
``paper_2405_04808_b200.configs.build_setup(1)``.  The full solution
(655,360 doubles) is not stored; the fixture keeps the iteration counts, the
residual history, the coarse-solve statistics and a fingerprint of the
solution (every 997th entry, its 2-norm and the norm of each variable kind),
so the GPU test can compare at full size without the reference.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

import tempokkt as tk  # noqa: E402
from tempokkt import krylov, multigrid  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    nx, nt, levels = 128, 1024, 4
    g = tk.TimeGrid(1.0, nt)
    p = tk.build_burgers(tk.BurgersConfig(nu=1e-2, alpha=0.1, n_elems=nx + 1,
                                          t_final=1.0, theta=1.0), g)
    x = (1.0 / (nx + 1)) * np.arange(1, nx + 1)
    p.u0 = np.where(x <= 0.5, np.sin(np.pi * x), 0.0)
    z = np.zeros((nt, nx))
    tr = tk.forward_solve(p, z, g)
    t0 = time.perf_counter()
    h = multigrid.build_hierarchy(p, tr.states, tr.states, z, g, levels, sweeps=1,
                                  cycle_kind="v", coarse_tol=1e-2)
    a = h.levels[0].kkt
    b = np.random.default_rng(1).standard_normal(a.dim)
    t1 = time.perf_counter()
    xs, rep = krylov.fgmres(a.as_operator(), multigrid.mg_preconditioner(h), b,
                            rel_tol=1e-8, max_iters=401)
    t2 = time.perf_counter()
    lay = a.layout
    kinds = {k: float(np.linalg.norm(xs[lay.rows(k)])) for k in ("u", "v", "z", "lam", "mu")}
    np.savez_compressed(
        os.path.join(HERE, "cfg1_full_solve.npz"),
        nx=nx, nt=nt, levels=levels, seed=1, rel_tol=1e-8, max_iters=401,
        fgmres_iters=rep.iterations, fgmres_hist=np.array(rep.residual_history),
        fgmres_rel=rep.final_relative_residual, coarse_calls=h.stats.calls,
        coarse_iters=h.stats.iters, b_norm=float(np.linalg.norm(b)),
        x_stride=997, x_sample=xs[::997], x_norm=float(np.linalg.norm(xs)),
        kind_names=np.array(list(kinds)), kind_norms=np.array(list(kinds.values())),
        fwd_state_sample=tr.states[::64, ::16],
        ref_setup_s=t1 - t0, ref_solve_s=t2 - t1)
    print("fgmres", rep.iterations, "rel", rep.final_relative_residual,
          "coarse", h.stats.calls, h.stats.iters, f"setup {t1 - t0:.1f}s solve {t2 - t1:.1f}s")


if __name__ == "__main__":
    main()
