"""Generate golden vectors by running the REAL reference package.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports ``tempokkt`` from /root/reference/pkg/src, builds small
instances of the reference's own problems plus reduced-size versions of
the BASELINE.json configurations, and records inputs/outputs of every
hot-path operation (stage Jacobians, Figure-3 operator apply, block
diagonal solve, block Jacobi, forward/backward/symmetric block
Gauss-Seidel, restriction/prolongation, coarse SGS-GMRES, V/F/W cycles
and full multigrid-preconditioned (F)GMRES solves with their iteration
counts and residual histories) into ``tests/golden/<case>.npz``.
Nothing on the GPU box reads /root/reference: the npz files travel.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

import tempokkt as tk  # noqa: E402
from tempokkt import kkt as tkkkt  # noqa: E402
from tempokkt import krylov, multigrid, smoothers, timedisc  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def vdp_spec(g, mu=1.0, alpha=0.1, n_controls=2, u0=(1.0, 1.0), theta=1.0):
    """Reference ProblemSpec for van der Pol; n_controls=1 puts the single
    control on the second equation (BASELINE configs 0/3)."""
    if n_controls == 2:
        return tk.build_vanderpol(tk.VanDerPolConfig(mu=mu, alpha=alpha,
                                                     u_init=tuple(u0)), g, theta=theta)
    fz = np.array([[0.0], [1.0]])
    return timedisc.ProblemSpec(
        n_u=2, n_z=1, mass=np.eye(2),
        f_eval=lambda u, z: np.array([u[1], mu * (1 - u[0] ** 2) * u[1] - u[0] + z[0]]),
        f_jac_u=lambda u, z: np.array([[0.0, 1.0],
                                       [-2 * mu * u[0] * u[1] - 1.0, mu * (1 - u[0] ** 2)]]),
        f_jac_z=lambda u, z: fz, u0=np.array(u0, dtype=np.float64), theta=theta,
        dt=g.dt, u_target=np.zeros((g.n_steps, 2)), z_target=np.zeros((g.n_steps, 1)),
        w_state=np.eye(2), w_control=alpha * np.eye(1), name="vdp1")


def burgers_spec(g, n_u, nu=1e-2, alpha=0.1, theta=0.5, u0_kind="step"):
    p = tk.build_burgers(tk.BurgersConfig(nu=nu, alpha=alpha, n_elems=n_u + 1,
                                          t_final=g.t_final, theta=theta), g)
    if u0_kind == "sinstep":
        x = (1.0 / (n_u + 1)) * np.arange(1, n_u + 1)
        p.u0 = np.where(x <= 0.5, np.sin(np.pi * x), 0.0)
    return p


def battery(name, p, g, u, v, z, levels, sweeps, seed, extra=None):
    """Record every hot-path operation on one linearisation point."""
    rng = np.random.default_rng(seed)
    out = dict(u=u, v=v, z=z, dt=g.dt, t_final=g.t_final, n=g.n_steps,
               levels=levels, sweeps=sweeps)
    st = tkkkt.build_stage_blocks(p, g.dt, u, v, z)
    out.update(K=st.k, C=st.c, B=st.b, Qu=st.q_u, Qv=st.q_v, Qz=st.q_z)
    a = tkkkt.assemble_kkt(st)
    ds = tkkkt.DiagonalSolver(a)
    x = rng.standard_normal(a.dim)
    b = rng.standard_normal(a.dim)
    out.update(x=x, b=b, Ax=a.apply(x), Dinv_b=ds.solve_all(b),
               jac1=smoothers.jacobi_apply(a, ds, b, x, 1),
               jac2=smoothers.jacobi_apply(a, ds, b, x, 2),
               fgs=smoothers.fgs_apply(a, ds, b, x),
               bgs=smoothers.bgs_apply(a, ds, b, x),
               sgs=smoothers.sgs_apply(a, ds, b, x),
               sgs0=smoothers.sgs_apply(a, ds, b, np.zeros(a.dim)))
    if levels > 1:
        h = multigrid.build_hierarchy(p, u, v, z, g, levels, sweeps=sweeps,
                                      cycle_kind="v", coarse_tol=1e-2)
        t0 = h.transfers[0]
        out["restrict_x"] = t0.restrict_kkt(x)
        xc = rng.standard_normal(t0.coarse_layout.dim)
        out["xc"] = xc
        out["prolong_xc"] = t0.prolong_kkt(xc)
        rc = rng.standard_normal(h.levels[-1].kkt.dim)
        out["coarse_r"] = rc
        out["coarse_x"] = multigrid.coarse_solve(h, rc)
        out["coarse_iters"] = h.stats.iters
        for kind in ("v", "w", "f"):
            h.cycle_kind = kind
            h.stats = multigrid.CoarseStats()
            out[f"cycle_{kind}"] = multigrid.cycle(h, 0, b)
            out[f"cycle_{kind}_coarse_iters"] = h.stats.iters
        h.cycle_kind = "v"
        for outer in ("fgmres", "gmres"):
            h.stats = multigrid.CoarseStats()
            fn = krylov.fgmres if outer == "fgmres" else krylov.gmres
            xs, rep = fn(a.as_operator(), multigrid.mg_preconditioner(h), b,
                         rel_tol=1e-8, max_iters=401)
            out[f"{outer}_x"] = xs
            out[f"{outer}_iters"] = rep.iterations
            out[f"{outer}_hist"] = np.array(rep.residual_history)
            out[f"{outer}_rel"] = rep.final_relative_residual
            out[f"{outer}_coarse_calls"] = h.stats.calls
            out[f"{outer}_coarse_iters"] = h.stats.iters
    if extra:
        out.update(extra)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, "dim", a.dim, {k: int(out[k]) for k in out if k.endswith("_iters")})


def main():
    rng = np.random.default_rng(1234)
    # 1. reference van der Pol (N_z = 2), backward Euler, perturbed iterate
    g = tk.TimeGrid(8.0, 32)
    p = vdp_spec(g)
    tr = tk.forward_solve(p, np.zeros((32, 2)), g)
    v = tr.states + 0.01 * rng.standard_normal(tr.states.shape)
    z = 0.1 * rng.standard_normal((32, 2))
    battery("vdp_ref", p, g, tr.states, v, z, levels=3, sweeps=2, seed=1,
            extra=dict(fwd_states=tr.states, mu=1.0, alpha=0.1, n_controls=2,
                       u0=np.array([1.0, 1.0]), theta=1.0))
    # 2. reference van der Pol, Crank-Nicolson (C_i varies with v)
    p = vdp_spec(g, theta=0.5)
    tr = tk.forward_solve(p, np.zeros((32, 2)), g)
    battery("vdp_cn", p, g, tr.states, v, z, levels=3, sweeps=1, seed=2,
            extra=dict(fwd_states=tr.states, mu=1.0, alpha=0.1, n_controls=2,
                       u0=np.array([1.0, 1.0]), theta=0.5))
    # 3. reference Burgers (step u0, Crank-Nicolson), perturbed iterate
    g = tk.TimeGrid(1.0, 32)
    p = burgers_spec(g, 16)
    tr = tk.forward_solve(p, np.zeros((32, 16)), g)
    v = tr.states + 0.01 * rng.standard_normal(tr.states.shape)
    z = 0.1 * rng.standard_normal((32, 16))
    battery("burgers_ref", p, g, tr.states, v, z, levels=3, sweeps=2, seed=3,
            extra=dict(fwd_states=tr.states, n_u=16, nu=1e-2, alpha=0.1, theta=0.5,
                       u0_kind="step"))
    # 4. BASELINE config 0 shape at full size: VdP N_z=1, u0=(1,0), T=5, nt=512
    T, n = 5.0, 512
    g = tk.TimeGrid(T, n)
    p = vdp_spec(g, n_controls=1, u0=(1.0, 0.0))
    t = g.dt * np.arange(1, n + 1)
    zc = (0.5 * np.sin(2 * np.pi * t / T)).reshape(n, 1)
    tr = tk.forward_solve(p, zc, g)
    battery("cfg0_vdp", p, g, tr.states, tr.states, zc, levels=3, sweeps=1, seed=0,
            extra=dict(fwd_states=tr.states, mu=1.0, alpha=0.1, n_controls=1,
                       u0=np.array([1.0, 0.0]), theta=1.0))
    # 5. BASELINE config 1 shape, reduced nx: Burgers nx=16, nt=64, BE, sin-step
    g = tk.TimeGrid(1.0, 64)
    p = burgers_spec(g, 16, theta=1.0, u0_kind="sinstep")
    tr = tk.forward_solve(p, np.zeros((64, 16)), g)
    battery("cfg1_burgers", p, g, tr.states, tr.states, np.zeros((64, 16)), levels=4,
            sweeps=1, seed=1,
            extra=dict(fwd_states=tr.states, n_u=16, nu=1e-2, alpha=0.1, theta=1.0,
                       u0_kind="sinstep"))


if __name__ == "__main__":
    main()
