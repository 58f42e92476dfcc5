"""Golden records at the BASELINE.json configuration SHAPES, by the REAL reference.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden_shapes.py [cfg2] [cfg3] [cfg4]

The full-size configs[2]/[3]/[4] are out of the reference's reach (its dense
per-interval inverses would need 16384 x 2560^2 doubles for configs[2]), so
each case keeps the configuration's spatial size, time step, hierarchy depth
(or the deepest the reduced nt allows) and solver, at the smallest nt that
keeps that depth:

* ``cfg2_shape``: Burgers nx=512 (interior nodes), nu=0.01, backward Euler,
  sin-step u0, z=0, dt = 1/16384 (configs[2]'s), nt=64, the 6-level V(1,1)
  hierarchy, rhs N(0,1) seed 2; one V-cycle and a <=60-iteration FGMRES.
* ``cfg3_shape``: van der Pol N_z=1, mu=1, u0=(1,0), dt = 2048/2^20,
  z(t) = 0.5 sin(2 pi t/50), nt=2^14, the 10-level V(1,1) hierarchy, rhs
  N(0,1) seed 3; one V-cycle and the full FGMRES (tol 1e-8, <=401 its).
* ``cfg4_shape``: Burgers nx=2048, nu=0.005, dt = 1/65536, smooth random
  8-mode control (seed 4), nt=4, 2 levels, rhs N(0,1) seed 4; operator apply,
  block-diagonal solve, one Jacobi sweep, one V-cycle and a <=30-iteration
  FGMRES -- pins the n_u=2048 local solves (2-CTA-cluster row kernel on the
  GPU) and the n_u=2048 coarse Gauss-Seidel chain to the reference.

Every case stores its linearisation point (u, v, z), so the GPU tests rebuild
the same hierarchy from the stored arrays without the reference.  Reference
code exercised: multigrid.py:190-301 (build_hierarchy, coarse_solve, cycle),
krylov.py:77-210 (fgmres), kkt.py:100-124, 228-247, 338-389, smoothers.py:61-76.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

import tempokkt as tk  # noqa: E402
from tempokkt import kkt as tkkkt  # noqa: E402
from tempokkt import krylov, multigrid, smoothers, timedisc  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def burgers_spec(g, n_u, nu, alpha=0.1, theta=1.0):
    p = tk.build_burgers(tk.BurgersConfig(nu=nu, alpha=alpha, n_elems=n_u + 1,
                                          t_final=g.t_final, theta=theta), g)
    x = (1.0 / (n_u + 1)) * np.arange(1, n_u + 1)
    p.u0 = np.where(x <= 0.5, np.sin(np.pi * x), 0.0)       # BASELINE sin-step u0
    return p


def vdp1_spec(g, mu=1.0, alpha=0.1, u0=(1.0, 0.0), theta=1.0):
    """van der Pol with the single control on the second equation."""
    fz = np.array([[0.0], [1.0]])
    return timedisc.ProblemSpec(
        n_u=2, n_z=1, mass=np.eye(2),
        f_eval=lambda u, z: np.array([u[1], mu * (1 - u[0] ** 2) * u[1] - u[0] + z[0]]),
        f_jac_u=lambda u, z: np.array([[0.0, 1.0],
                                       [-2 * mu * u[0] * u[1] - 1.0, mu * (1 - u[0] ** 2)]]),
        f_jac_z=lambda u, z: fz, u0=np.array(u0, dtype=np.float64), theta=theta,
        dt=g.dt, u_target=np.zeros((g.n_steps, 2)), z_target=np.zeros((g.n_steps, 1)),
        w_state=np.eye(2), w_control=alpha * np.eye(1), name="vdp1")


def fourier_control(nt, dt, nx, modes=8, std=0.1, seed=4):
    """Smooth random control sum_k c_k cos(pi k t/T) sin(pi k x), c ~ N(0, std)."""
    t = dt * np.arange(1, nt + 1)
    x = np.arange(1, nx + 1) / (nx + 1.0)
    c = np.random.default_rng(seed).normal(0.0, std, size=modes)
    k = np.arange(1, modes + 1)
    sx = np.sin(np.pi * k[:, None] * x[None, :])
    ct = np.cos(np.pi * k[None, :] * t[:, None] / (nt * dt))
    return (ct * c[None, :]) @ sx


def record(name, p, g, u, v, z, levels, seed, fgmres_its, extra=None, ops=False):
    t0 = time.perf_counter()
    h = multigrid.build_hierarchy(p, u, v, z, g, levels, sweeps=1, cycle_kind="v",
                                  coarse_tol=1e-2)
    t1 = time.perf_counter()
    a = h.levels[0].kkt
    b = np.random.default_rng(seed).standard_normal(a.dim)
    out = dict(u=u, v=v, z=z, dt=g.dt, t_final=g.t_final, n=g.n_steps, levels=levels,
               sweeps=1, seed=seed, b=b, fgmres_max_iters=fgmres_its)
    if ops:
        rng = np.random.default_rng(seed + 100)
        x = rng.standard_normal(a.dim)
        ds = h.levels[0].dsolve
        out.update(x=x, Ax=a.apply(x), Dinv_b=ds.solve_all(b),
                   jac1=smoothers.jacobi_apply(a, ds, b, x, 1))
    h.stats = multigrid.CoarseStats()
    out["cycle_v"] = multigrid.cycle(h, 0, b)
    out["cycle_v_coarse_iters"] = h.stats.iters
    h.stats = multigrid.CoarseStats()
    t2 = time.perf_counter()
    xs, rep = krylov.fgmres(a.as_operator(), multigrid.mg_preconditioner(h), b,
                            rel_tol=1e-8, max_iters=fgmres_its)
    t3 = time.perf_counter()
    out.update(fgmres_x=xs, fgmres_iters=rep.iterations,
               fgmres_hist=np.array(rep.residual_history), fgmres_rel=rep.final_relative_residual,
               fgmres_coarse_calls=h.stats.calls, fgmres_coarse_iters=h.stats.iters,
               ref_setup_s=t1 - t0, ref_solve_s=t3 - t2)
    if extra:
        out.update(extra)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, "dim", a.dim, "levels", levels, "cycle coarse its", out["cycle_v_coarse_iters"],
          "fgmres", rep.iterations, "rel", rep.final_relative_residual,
          "coarse", h.stats.calls, h.stats.iters,
          f"setup {t1 - t0:.1f}s solve {t3 - t2:.1f}s", flush=True)


def cfg2():
    nx, nt, levels = 512, 64, 6
    dt = 1.0 / 16384
    g = tk.TimeGrid(nt * dt, nt)
    p = burgers_spec(g, nx, nu=0.01)
    z = np.zeros((nt, nx))
    u = tk.forward_solve(p, z, g).states
    record("cfg2_shape", p, g, u, u, z, levels, seed=2, fgmres_its=60, ops=True,
           extra=dict(n_u=nx, nu=0.01, alpha=0.1, theta=1.0, u0_kind="sinstep"))


def cfg3():
    nt, levels = 1 << 14, 10
    dt = 2048.0 / (1 << 20)
    g = tk.TimeGrid(nt * dt, nt)
    p = vdp1_spec(g)
    t = dt * np.arange(1, nt + 1)
    z = (0.5 * np.sin(2 * np.pi * t / 50.0)).reshape(nt, 1)
    u = tk.forward_solve(p, z, g).states
    record("cfg3_shape", p, g, u, u, z, levels, seed=3, fgmres_its=401,
           extra=dict(mu=1.0, alpha=0.1, n_controls=1, u0=np.array([1.0, 0.0]), theta=1.0))


def cfg4():
    nx, nt, levels = 2048, 4, 2
    dt = 1.0 / 65536
    g = tk.TimeGrid(nt * dt, nt)
    p = burgers_spec(g, nx, nu=0.005)
    z = fourier_control(nt, dt, nx)
    u = tk.forward_solve(p, z, g).states
    record("cfg4_shape", p, g, u, u, z, levels, seed=4, fgmres_its=30, ops=True,
           extra=dict(n_u=nx, nu=0.005, alpha=0.1, theta=1.0, u0_kind="sinstep"))


if __name__ == "__main__":
    which = sys.argv[1:] or ["cfg2", "cfg3", "cfg4"]
    for w in which:
        globals()[w]()
