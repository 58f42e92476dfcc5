"""Problem builders: van der Pol (problems.py:24-97), 1D viscous Burgers with
P1 finite elements (problems.py:100-197) and Neumann boundary control of the
1D heat equation (problems.py:200-266; general dense stage blocks).

Each returns a :class:`ProblemSpec` with the reference's Python callables
(so generic code paths and tests can evaluate F) plus a ``native`` tag that
routes the forward march and the stage linearisation to
libtempokkt_b200.so.  Extra knobs (``n_controls``, ``u0_kind``) express the
BASELINE.json configurations; their defaults reproduce the reference.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .timedisc import ProblemSpec, TimeGrid, forward_solve


@dataclass
class VanDerPolConfig:
    mu: float = 1.0
    alpha: float = 0.1
    t_final: float = 8.0
    data_mu: float = 0.01
    u_init: tuple = (1.0, 1.0)
    n_controls: int = 2          # 2: F_z = I (reference); 1: control on the 2nd equation

    def __post_init__(self):
        if self.alpha <= 0.0:
            raise ValueError("alpha must be positive")
        if self.t_final <= 0.0:
            raise ValueError("t_final must be positive")
        if self.n_controls not in (1, 2):
            raise ValueError("n_controls must be 1 or 2")


def _vdp_callables(mu, nc):
    fz = np.eye(2) if nc == 2 else np.array([[0.0], [1.0]])

    def f_eval(u, z):
        z0 = z[0] if nc == 2 else 0.0
        z1 = z[1] if nc == 2 else z[0]
        return np.array([u[1] + z0, mu * (1.0 - u[0] ** 2) * u[1] - u[0] + z1])

    def f_jac_u(u, z):
        return np.array([[0.0, 1.0],
                         [-2.0 * mu * u[0] * u[1] - 1.0, mu * (1.0 - u[0] ** 2)]])

    def f_jac_z(u, z):
        return fz

    def f_hess_vec(u, z, lam, du):
        h = lam[1] * np.array([[-2.0 * mu * u[1], -2.0 * mu * u[0]],
                               [-2.0 * mu * u[0], 0.0]])
        return h @ du

    return f_eval, f_jac_u, f_jac_z, f_hess_vec


def build_vanderpol(cfg: VanDerPolConfig, g: TimeGrid, theta: float = 1.0,
                    with_targets: bool = True) -> ProblemSpec:
    """Two-state oscillator; tracking data from the same oscillator with
    damping ``data_mu`` at zero control (problems.py:42-97)."""
    nc = cfg.n_controls
    u0 = np.array(cfg.u_init, dtype=np.float64)
    fe, fu, fz, fh = _vdp_callables(cfg.mu, nc)
    n = g.n_steps
    u_target = np.zeros((n, 2))
    if with_targets:
        fe_d, fu_d, _, _ = _vdp_callables(cfg.data_mu, nc)
        data = ProblemSpec(n_u=2, n_z=nc, mass=np.eye(2), f_eval=fe_d, f_jac_u=fu_d,
                           f_jac_z=fz, u0=u0, theta=theta, dt=g.dt,
                           u_target=np.zeros((n, 2)), z_target=np.zeros((n, nc)),
                           w_state=np.eye(2), w_control=cfg.alpha * np.eye(nc),
                           native={"kind": "vanderpol", "mu": cfg.data_mu})
        u_target = forward_solve(data, np.zeros((n, nc)), g).states
    return ProblemSpec(n_u=2, n_z=nc, mass=np.eye(2), f_eval=fe, f_jac_u=fu, f_jac_z=fz,
                       u0=u0, theta=theta, dt=g.dt, u_target=u_target,
                       z_target=np.zeros((n, nc)), w_state=np.eye(2),
                       w_control=cfg.alpha * np.eye(nc), f_hess_vec=fh, name="vanderpol",
                       native={"kind": "vanderpol", "mu": cfg.mu})


@dataclass
class BurgersConfig:
    nu: float = 1e-2
    alpha: float = 0.1
    n_elems: int = 128
    t_final: float = 1.0
    theta: float = 0.5
    u0_kind: str = "step"        # "step" (reference) or "sinstep" (BASELINE: sin(pi x), x<=0.5)

    def __post_init__(self):
        if self.nu <= 0.0:
            raise ValueError("nu must be positive")
        if self.n_elems < 3:
            raise ValueError("n_elems must be >= 3")
        if self.u0_kind not in ("step", "sinstep"):
            raise ValueError("u0_kind must be 'step' or 'sinstep'")


def tridiag(n, lo, di, hi):
    a = np.zeros((n, n))
    a[np.arange(n), np.arange(n)] = di
    a[np.arange(1, n), np.arange(n - 1)] = lo
    a[np.arange(n - 1), np.arange(1, n)] = hi
    return a


def burgers_convection(u):
    up = np.concatenate([u[1:], [0.0]])
    um = np.concatenate([[0.0], u[:-1]])
    return (up * up + u * up - u * um - um * um) / 6.0


def burgers_convection_jac(u):
    n = u.shape[0]
    up = np.concatenate([u[1:], [0.0]])
    um = np.concatenate([[0.0], u[:-1]])
    return tridiag(n, (-u[1:] - 2.0 * u[:-1]) / 6.0, (up - um) / 6.0,
                   (2.0 * u[1:] + u[:-1]) / 6.0)


def build_burgers(cfg: BurgersConfig, g: TimeGrid) -> ProblemSpec:
    """P1 FE semi-discretisation, interior nodes only, N_z = N_u
    (problems.py:149-197)."""
    n = cfg.n_elems - 1
    h = 1.0 / cfg.n_elems
    mass = tridiag(n, h / 6.0, 4.0 * h / 6.0, h / 6.0)
    stiff = tridiag(n, -1.0 / h, 2.0 / h, -1.0 / h)
    nu = cfg.nu

    def f_eval(u, z):
        return -nu * (stiff @ u) - burgers_convection(u) + mass @ z

    def f_jac_u(u, z):
        return -nu * stiff - burgers_convection_jac(u)

    def f_jac_z(u, z):
        return mass

    def f_hess_vec(u, z, lam, du):
        lam_p = np.concatenate([lam[1:], [0.0]])
        lam_m = np.concatenate([[0.0], lam[:-1]])
        diag = (lam_m - lam_p) / 3.0
        off = (lam[:-1] - lam[1:]) / 6.0
        out = diag * du
        out[:-1] += off * du[1:]
        out[1:] += off * du[:-1]
        return -out

    x = h * np.arange(1, n + 1)
    step = np.where(x <= 0.5, 1.0, 0.0)
    u0 = step.copy() if cfg.u0_kind == "step" else np.where(x <= 0.5, np.sin(np.pi * x), 0.0)
    return ProblemSpec(n_u=n, n_z=n, mass=mass, f_eval=f_eval, f_jac_u=f_jac_u,
                       f_jac_z=f_jac_z, u0=u0, theta=cfg.theta, dt=g.dt,
                       u_target=np.broadcast_to(step, (g.n_steps, n)),
                       z_target=np.broadcast_to(np.zeros(n), (g.n_steps, n)), w_state=mass,
                       w_control=cfg.alpha * mass, f_hess_vec=f_hess_vec, name="burgers",
                       native={"kind": "burgers", "nu": nu})


@dataclass
class HeatNeumannConfig:
    """Left-flux boundary control of the 1D heat equation (problems.py:200-215):
    tracking weights alpha1 (running) and alpha2 (terminal), n_cells P1 cells."""

    alpha1: float = 1e3
    alpha2: float = 0.0
    n_cells: int = 16
    t_final: float = 1.0

    def __post_init__(self):
        if self.alpha1 < 0.0 or self.alpha2 < 0.0:
            raise ValueError("tracking weights must be nonnegative")
        if self.alpha1 == 0.0 and self.alpha2 == 0.0:
            raise ValueError("alpha1 and alpha2 cannot both be zero")


def build_heat_neumann(cfg: HeatNeumannConfig, g: TimeGrid, theta: float = 1.0) -> ProblemSpec:
    """P1 FE heat operator on [0, 1] with flux boundary data, every node an
    unknown (problems.py:218-266): F(u, z) = -A u - z e_first with the Neumann
    mass / stiffness matrices, u0 = cos(pi x), zero targets, w_state =
    alpha1 M, scalar control weight 1.  N_z = 1, N_u = n_cells + 1: general
    dense stage blocks (the warp-per-row kernels of tk_denseg.cu)."""
    nn = cfg.n_cells + 1
    h = 1.0 / cfg.n_cells
    mass = tridiag(nn, h / 6.0, 4.0 * h / 6.0, h / 6.0)
    stiff = tridiag(nn, -1.0 / h, 2.0 / h, -1.0 / h)
    for a, corner in ((mass, h / 3.0), (stiff, 1.0 / h)):
        a[0, 0] = corner
        a[-1, -1] = corner
    fz = np.zeros((nn, 1))
    fz[0, 0] = -1.0                       # -z * e_first

    def f_eval(u, z):
        return -stiff @ u + fz[:, 0] * z[0]

    def f_jac_u(u, z):
        return -stiff

    def f_jac_z(u, z):
        return fz

    return ProblemSpec(
        n_u=nn, n_z=1, mass=mass, f_eval=f_eval, f_jac_u=f_jac_u, f_jac_z=f_jac_z,
        u0=np.cos(np.pi * h * np.arange(nn)), theta=theta, dt=g.dt,
        u_target=np.zeros((g.n_steps, nn)), z_target=np.zeros((g.n_steps, 1)),
        w_state=cfg.alpha1 * mass, w_control=np.array([[1.0]]),
        w_terminal=(cfg.alpha2 * mass) if cfg.alpha2 > 0.0 else None, name="heat-neumann")
