"""Golden record of the reference's heat-Neumann problem (general dense stage
blocks: N_z = 1 boundary control, N_u = n_cells + 1), by the REAL reference
(run in the build container, the only place /root/reference exists):

    python tests/golden/make_golden_heat.py

n_cells = 16 (n_u = 17), backward Euler, T = 1, N = 32, 3 levels, one sweep;
the linearisation point is stored, so the GPU test rebuilds the hierarchy
without the reference.  Reference code exercised: problems.py:218-266,
kkt.py:100-124, 228-247, 338-389, smoothers.py:61-152, multigrid.py:104-132,
190-301, krylov.py:77-210.
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import tempokkt as tk  # noqa: E402
from tempokkt import kkt as K, krylov, multigrid, smoothers  # noqa: E402
from tempokkt.problems import HeatNeumannConfig, build_heat_neumann  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    n, levels = 32, 3
    g = tk.TimeGrid(1.0, n)
    p = build_heat_neumann(HeatNeumannConfig(n_cells=16), g)
    rng = np.random.default_rng(21)
    z = 0.5 * rng.standard_normal((n, 1))
    u = tk.forward_solve(p, z, g).states
    v = u + 0.01 * rng.standard_normal(u.shape)
    st = K.build_stage_blocks(p, g.dt, u, v, z)
    a = K.assemble_kkt(st)
    ds = K.DiagonalSolver(a)
    dim = a.layout.dim
    x, b = rng.standard_normal(dim), rng.standard_normal(dim)
    h = multigrid.build_hierarchy(p, u, v, z, g, levels, sweeps=1, coarse_tol=1e-2)
    t = h.transfers[0]
    xc = rng.standard_normal(t.coarse_layout.dim)
    cyc = multigrid.cycle(h, 0, b)
    its_cycle = h.stats.iters if hasattr(h, "stats") else -1
    xs, rep = krylov.fgmres(a.as_operator(), multigrid.mg_preconditioner(h), b, rel_tol=1e-8,
                            max_iters=40)
    np.savez_compressed(
        os.path.join(HERE, "heat_ref.npz"), n=n, levels=levels, n_cells=16, u=u, v=v, z=z, x=x, b=b,
        k0=st.k[0], c1=st.c[1], b0=st.b[0], q_u0=st.q_u[0], q_z0=st.q_z[0],
        apply=a.apply(x), solve_all=ds.solve_all(b),
        jacobi2=smoothers.jacobi_apply(a, ds, b, x.copy(), 2, 1.0),
        jacobi_w=smoothers.jacobi_apply(a, ds, b, x.copy(), 1, 0.7),
        fgs=smoothers.fgs_apply(a, ds, b, x.copy()), bgs=smoothers.bgs_apply(a, ds, b, x.copy()),
        sgs=smoothers.sgs_apply(a, ds, b, x.copy()),
        restrict=t.restrict_kkt(x), prolong_xc=t.prolong_kkt(xc), xc=xc,
        cycle=cyc, fgmres_x=xs, fgmres_iters=rep.iterations,
        fgmres_hist=np.array(rep.residual_history))
    print("heat_ref.npz dim", dim, "fgmres its", rep.iterations, "converged", rep.converged)


if __name__ == "__main__":
    main()
