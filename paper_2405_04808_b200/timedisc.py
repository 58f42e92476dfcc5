"""Time grids, problem contract, theta-method forward march and stage weights.

Mirrors the reference module timedisc.py (TimeGrid :35-58, ProblemSpec
:61-94, Trajectory :97-102, theta_residual :112, stage_blocks :133,
forward_solve :152, stage_weights :194).  ``ProblemSpec`` additionally
carries an optional ``native`` descriptor naming a built-in problem
(van der Pol, Burgers) whose forward march and stage linearisation then run
in libtempokkt_b200.so; specs without it use the Python callables (setup
only -- the hot path is always the CUDA kernels).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from . import _lib
from .errors import DimensionMismatch, NewtonDivergence, NonFiniteValue

NEWTON_MAX_ITERS = 25


@dataclass(frozen=True)
class TimeGrid:
    """Uniform partition of [0, t_final] into n_steps intervals."""

    t_final: float
    n_steps: int

    def __post_init__(self):
        if self.n_steps < 1:
            raise ValueError("n_steps must be >= 1")
        if self.t_final <= 0.0:
            raise ValueError("t_final must be positive")

    @property
    def dt(self) -> float:
        return self.t_final / self.n_steps

    def node(self, i: int) -> float:
        return i * self.dt

    def coarsened(self) -> "TimeGrid":
        if self.n_steps % 2 != 0:
            raise ValueError("cannot coarsen an odd step count")
        return TimeGrid(self.t_final, self.n_steps // 2)


@dataclass
class ProblemSpec:
    """``M du/dt = F(u, z)``, ``u(0) = u0`` plus tracking data and weights."""

    n_u: int
    n_z: int
    mass: np.ndarray
    f_eval: Callable
    f_jac_u: Callable
    f_jac_z: Callable
    u0: np.ndarray
    theta: float
    dt: float
    u_target: np.ndarray
    z_target: np.ndarray
    w_state: np.ndarray
    w_control: np.ndarray
    w_terminal: Optional[np.ndarray] = None
    f_hess_vec: Optional[Callable] = None
    name: str = "problem"
    native: Optional[dict] = None

    @property
    def n_steps(self) -> int:
        return self.u_target.shape[0]


@dataclass
class Trajectory:
    states: np.ndarray
    controls: np.ndarray


def theta_residual(p: ProblemSpec, v_i, u_next, z_next, dt: float) -> np.ndarray:
    """``-M u_next + M v_i + dt*theta*F(u_next,z) + dt*(1-theta)*F(v_i,z)``."""
    v_i = np.asarray(v_i, dtype=np.float64)
    u_next = np.asarray(u_next, dtype=np.float64)
    z_next = np.asarray(z_next, dtype=np.float64)
    if v_i.shape != (p.n_u,) or u_next.shape != (p.n_u,) or z_next.shape != (p.n_z,):
        raise DimensionMismatch("stage vector has wrong dimension")
    th = p.theta
    r = p.mass @ (v_i - u_next)
    if th != 0.0:
        r = r + dt * th * p.f_eval(u_next, z_next)
    if th != 1.0:
        r = r + dt * (1.0 - th) * p.f_eval(v_i, z_next)
    if not np.isfinite(r).all():
        raise NonFiniteValue("non-finite stage residual")
    return r


def stage_jacobians(p: ProblemSpec, v_i, u_next, z_next, dt: float):
    """Dense (K, C, B) of one stage from the Python callables."""
    th = p.theta
    k = -p.mass + dt * th * p.f_jac_u(u_next, z_next)
    c = p.mass + dt * (1.0 - th) * p.f_jac_u(v_i, z_next)
    b = dt * th * p.f_jac_z(u_next, z_next) + dt * (1.0 - th) * p.f_jac_z(v_i, z_next)
    return k, c, b


def stage_weights(p: ProblemSpec, dt: float, i: int, n_steps: int):
    """(Q_u, Q_v, Q_z) of stage i: 0.5*dt*w_state (+0.5*w_terminal at the
    last stage), and dt*w_control."""
    q_u = 0.5 * dt * p.w_state
    q_z = dt * p.w_control
    if p.w_terminal is not None and i == n_steps - 1:
        q_u = q_u + 0.5 * p.w_terminal
    return q_u, q_u.copy(), q_z


def _native_forward(p: ProblemSpec, controls: np.ndarray, grid: TimeGrid, tol: float):
    nat = getattr(p, "native", None)
    n = grid.n_steps
    lib = _lib.load()
    states = np.empty((n, p.n_u))
    u0 = np.ascontiguousarray(p.u0, dtype=np.float64)
    z = np.ascontiguousarray(controls, dtype=np.float64)
    if nat["kind"] == "vanderpol":
        rc = lib.tk_forward_vanderpol_host(n, grid.dt, p.theta, nat["mu"], p.n_z,
                                           u0.ctypes.data, z.ctypes.data, tol,
                                           states.ctypes.data)
    elif nat["kind"] == "burgers":
        rc = lib.tk_forward_burgers_host(n, p.n_u, grid.dt, p.theta, nat["nu"],
                                         u0.ctypes.data, z.ctypes.data, tol,
                                         states.ctypes.data)
    else:
        raise ValueError(f"unknown native problem {nat['kind']!r}")
    if rc == _lib.TK_ERR_NEWTON:
        raise NewtonDivergence("forward march: Newton failed to converge")
    _lib.check(rc, "forward_solve")
    return states


def forward_solve(p: ProblemSpec, controls, grid: TimeGrid,
                  newton_tol: float = 1e-12) -> Trajectory:
    """Nonlinear theta-method march from p.u0 (timedisc.py:152-191)."""
    controls = np.asarray(controls, dtype=np.float64)
    n = grid.n_steps
    if controls.shape != (n, p.n_z):
        raise DimensionMismatch(f"controls shape {controls.shape} != ({n}, {p.n_z})")
    if getattr(p, "native", None) is not None:       # reference specs have no tag
        return Trajectory(states=_native_forward(p, controls, grid, newton_tol),
                          controls=controls.copy())
    # generic specs: per-step Newton with the callables (setup path only)
    import scipy.linalg
    dt = grid.dt
    states = np.empty((n, p.n_u))
    u_prev = np.array(p.u0, dtype=np.float64)
    for i in range(n):
        z = controls[i]
        u = u_prev.copy()
        tol = newton_tol * np.linalg.norm(p.mass @ u_prev) + newton_tol
        for _ in range(NEWTON_MAX_ITERS):
            r = theta_residual(p, u_prev, u, z, dt)
            if np.linalg.norm(r) <= tol:
                break
            k, _, _ = stage_jacobians(p, u_prev, u, z, dt)
            u = u - scipy.linalg.lu_solve(scipy.linalg.lu_factor(k), r)
        else:
            r = theta_residual(p, u_prev, u, z, dt)
            if np.linalg.norm(r) > tol:
                raise NewtonDivergence(f"step {i + 1}: Newton did not converge")
        states[i] = u
        u_prev = u
    return Trajectory(states=states, controls=controls.copy())
