"""The BASELINE.json configurations as reproducible setups.

configs[0]  van der Pol, N_z=1, mu=1, T=5, nt=512, z(t)=0.5 sin(2 pi t/T), 3-level V(1,1)
configs[1]  Burgers nx=128, nu=0.01, T=1, nt=1024, BE, sin-step u0, z=0, 4-level V
configs[2]  Burgers nx=512, nt=16384, seed 2, 6-level V          (time slabs over 1/2/4/8 GPUs)
configs[3]  van der Pol nt=2^20, T=2048, z(t)=0.5 sin(2 pi t/50), seed 3, 10-level V
configs[4]  Burgers nx=2048, nt=65536, nu=0.005, smooth random 8-mode control, 8-level V

"nx" counts interior nodes (= N_u = N_z), i.e. nx+1 linear elements.  The
linearisation point is the forward march under the stated control (u = v);
the right-hand side is i.i.d. N(0,1) in fp64 from ``numpy.random.default_rng(seed)``
over the whole KKT dimension N*(4 N_u + N_z).  Solver: (F)GMRES tol 1e-8,
V-cycle with 1 pre- and 1 post-sweep of block Jacobi, coarse SGS-GMRES at
the reference's default tolerance 1e-2 (multigrid.py:167).  Controls are
sampled at the interval end points t_i = i*dt (i = 1..N) where the reference
indexes z_i (timedisc.py:6-8).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .problems import BurgersConfig, VanDerPolConfig, build_burgers, build_vanderpol
from .timedisc import ProblemSpec, TimeGrid, forward_solve

CONFIGS = {
    0: dict(problem="vanderpol", mu=1.0, alpha=0.1, n_controls=1, u0=(1.0, 0.0), t_final=5.0,
            nt=512, theta=1.0, control=("sin", 5.0), seed=0, levels=3),
    1: dict(problem="burgers", nx=128, nu=0.01, alpha=0.1, t_final=1.0, nt=1024, theta=1.0,
            u0_kind="sinstep", control=("zero",), seed=1, levels=4),
    2: dict(problem="burgers", nx=512, nu=0.01, alpha=0.1, t_final=1.0, nt=16384, theta=1.0,
            u0_kind="sinstep", control=("zero",), seed=2, levels=6),
    3: dict(problem="vanderpol", mu=1.0, alpha=0.1, n_controls=1, u0=(1.0, 0.0),
            t_final=2048.0, nt=1 << 20, theta=1.0, control=("sin", 50.0), seed=3, levels=10),
    4: dict(problem="burgers", nx=2048, nu=0.005, alpha=0.1, t_final=1.0, nt=65536, theta=1.0,
            u0_kind="sinstep", control=("fourier", 8, 0.1), seed=4, levels=8),
}
SOLVER = dict(sweeps=1, omega=1.0, cycle="v", coarse_tol=1e-2, coarse_max_iters=401,
              rel_tol=1e-8, max_iters=401)


@dataclass
class Setup:
    index: int
    params: dict
    problem: ProblemSpec
    grid: TimeGrid
    u: np.ndarray
    v: np.ndarray
    z: np.ndarray
    levels: int
    solver: dict = field(default_factory=lambda: dict(SOLVER))

    @property
    def n_u(self):
        return self.problem.n_u

    @property
    def n_z(self):
        return self.problem.n_z

    @property
    def dim(self):
        return self.grid.n_steps * (4 * self.n_u + self.n_z)

    @property
    def dof_per_step(self):
        return 4 * self.n_u + self.n_z

    def rhs(self) -> np.ndarray:
        return np.random.default_rng(self.params["seed"]).standard_normal(self.dim)

    def describe(self) -> str:
        p = self.params
        if p["problem"] == "vanderpol":
            return f"vanderpol_nz{p['n_controls']}_nt{self.grid.n_steps}_L{self.levels}"
        return f"burgers_nx{p['nx']}_nt{self.grid.n_steps}_L{self.levels}"


def _controls(p, grid: TimeGrid, n_z: int, x=None) -> np.ndarray:
    n = grid.n_steps
    t = grid.dt * np.arange(1, n + 1)
    kind = p["control"][0]
    if kind == "zero":
        return np.zeros((n, n_z))
    if kind == "sin":
        period = p["control"][1]
        return (0.5 * np.sin(2.0 * np.pi * t / period)).reshape(n, 1).repeat(n_z, axis=1)
    if kind == "fourier":
        modes, std = p["control"][1], p["control"][2]
        c = np.random.default_rng(p["seed"]).normal(0.0, std, size=modes)
        k = np.arange(1, modes + 1)
        sx = np.sin(np.pi * k[:, None] * x[None, :])                 # (modes, nx)
        ct = np.cos(np.pi * k[None, :] * t[:, None] / grid.t_final)  # (n, modes)
        return (ct * c[None, :]) @ sx
    raise ValueError(f"unknown control {kind!r}")


def build_setup(index: int, nt: int = None, nx: int = None, levels: int = None,
                seed: int = None) -> Setup:
    """Build configs[index] (optionally with reduced nt / nx / levels for
    parity tests at oracle-sized problems)."""
    p = dict(CONFIGS[index])
    if nt is not None:
        p["nt"] = nt
    if nx is not None:
        p["nx"] = nx
    if seed is not None:
        p["seed"] = seed
    L = p["levels"] if levels is None else levels
    grid = TimeGrid(p["t_final"], p["nt"])
    if p["problem"] == "vanderpol":
        cfg = VanDerPolConfig(mu=p["mu"], alpha=p["alpha"], t_final=p["t_final"],
                              u_init=tuple(p["u0"]), n_controls=p["n_controls"])
        prob = build_vanderpol(cfg, grid, theta=p["theta"], with_targets=False)
        z = _controls(p, grid, prob.n_z)
    else:
        cfg = BurgersConfig(nu=p["nu"], alpha=p["alpha"], n_elems=p["nx"] + 1,
                            t_final=p["t_final"], theta=p["theta"], u0_kind=p["u0_kind"])
        prob = build_burgers(cfg, grid)
        xs = np.arange(1, p["nx"] + 1) / (p["nx"] + 1.0)
        z = _controls(p, grid, prob.n_z, xs)
    traj = forward_solve(prob, z, grid)
    return Setup(index=index, params=p, problem=prob, grid=grid, u=traj.states,
                 v=traj.states, z=z, levels=L)
