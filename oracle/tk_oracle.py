"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

This module is a plain numpy restatement of the reference package
``tempokkt`` (arXiv 2405.04808 artifact, mounted read-only at
/root/reference/pkg/src/tempokkt) for the data-parallel hot path:
stage linearisation, the Figure-3 block-tridiagonal augmented (KKT)
operator, its explicit block-diagonal inverse, block Jacobi / forward /
backward / symmetric block Gauss-Seidel, the time-level transfers, the
rediscretised hierarchy, V/F/W cycles, the SGS-preconditioned GMRES
coarse solve and right-preconditioned (F)GMRES.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it, and only as
the checker / the timed CPU reference -- never as the product path.

Pinning: every function is checked against golden vectors produced by
running the real reference in this container
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``), see
``tests/test_oracle_golden.py``.  Citations are ``file:line`` inside
/root/reference/pkg/src/tempokkt/.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np
import scipy.linalg

PIVOT_FLOOR = 1e-14            # linalg.py:38
BREAKDOWN_TOL = 1e-14          # krylov.py:29
NEWTON_MAX_ITERS = 25          # timedisc.py:32


# --------------------------------------------------------------------------
# problems (problems.py) -- only what the hot path consumes
# --------------------------------------------------------------------------
@dataclass
class Problem:
    """Semi-discrete dynamics ``M du/dt = F(u, z)`` (timedisc.py:61-94)."""
    n_u: int
    n_z: int
    mass: np.ndarray
    f: Callable
    f_u: Callable
    f_z: Callable
    u0: np.ndarray
    theta: float
    w_state: np.ndarray
    w_control: np.ndarray
    w_terminal: Optional[np.ndarray] = None


def vanderpol(mu=1.0, alpha=0.1, n_controls=2, u0=(1.0, 1.0), theta=1.0) -> Problem:
    """van der Pol oscillator (problems.py:42-97).  ``n_controls=2`` is the
    reference's F_z = I; ``n_controls=1`` is the single control entering the
    second equation (BASELINE configs 0 and 3)."""
    def f(u, z):
        zz = (z[0], z[1]) if n_controls == 2 else (0.0, z[0])
        return np.array([u[1] + zz[0], mu * (1.0 - u[0] ** 2) * u[1] - u[0] + zz[1]])

    def f_u(u, z):
        return np.array([[0.0, 1.0],
                         [-2.0 * mu * u[0] * u[1] - 1.0, mu * (1.0 - u[0] ** 2)]])

    fz = np.eye(2) if n_controls == 2 else np.array([[0.0], [1.0]])
    return Problem(n_u=2, n_z=n_controls, mass=np.eye(2), f=f, f_u=f_u,
                   f_z=lambda u, z: fz, u0=np.array(u0, dtype=np.float64),
                   theta=theta, w_state=np.eye(2),
                   w_control=alpha * np.eye(n_controls))


def _tridiag(n, lo, di, hi):
    a = np.zeros((n, n))
    a[np.arange(n), np.arange(n)] = di
    a[np.arange(1, n), np.arange(n - 1)] = lo
    a[np.arange(n - 1), np.arange(1, n)] = hi
    return a


def burgers_convection(u):
    """Galerkin convection vector (problems.py:119-124)."""
    up = np.concatenate([u[1:], [0.0]])
    um = np.concatenate([[0.0], u[:-1]])
    return (up * up + u * up - u * um - um * um) / 6.0


def burgers_convection_jac(u):
    """Its Jacobian (problems.py:127-138)."""
    n = u.shape[0]
    up = np.concatenate([u[1:], [0.0]])
    um = np.concatenate([[0.0], u[:-1]])
    return _tridiag(n, (-u[1:] - 2.0 * u[:-1]) / 6.0, (up - um) / 6.0,
                    (2.0 * u[1:] + u[:-1]) / 6.0)


def burgers(n_u=127, nu=1e-2, alpha=0.1, theta=0.5, u0_kind="step") -> Problem:
    """1D viscous Burgers, P1 finite elements, interior nodes only
    (problems.py:149-197).  ``n_u`` interior nodes => ``n_u + 1`` elements.
    ``u0_kind='step'`` is the reference's initial step; ``'sinstep'`` is
    BASELINE's ``sin(pi x)`` for x <= 0.5, else 0."""
    n = n_u
    h = 1.0 / (n + 1)
    mass = _tridiag(n, h / 6.0, 4.0 * h / 6.0, h / 6.0)
    stiff = _tridiag(n, -1.0 / h, 2.0 / h, -1.0 / h)
    x = h * np.arange(1, n + 1)
    if u0_kind == "step":
        u0 = np.where(x <= 0.5, 1.0, 0.0)
    else:
        u0 = np.where(x <= 0.5, np.sin(np.pi * x), 0.0)
    return Problem(
        n_u=n, n_z=n, mass=mass,
        f=lambda u, z: -nu * (stiff @ u) - burgers_convection(u) + mass @ z,
        f_u=lambda u, z: -nu * stiff - burgers_convection_jac(u),
        f_z=lambda u, z: mass, u0=u0, theta=theta,
        w_state=mass, w_control=alpha * mass)


def heat_neumann(n_cells=16, alpha1=1e3, alpha2=0.0, theta=1.0) -> Problem:
    """Neumann boundary control of the 1D heat equation (problems.py:200-266):
    P1 finite elements on n_cells cells, every node an unknown, the scalar
    control is the left boundary flux, F(u, z) = -A u - z e_first."""
    nn = n_cells + 1
    h = 1.0 / n_cells
    mass = _tridiag(nn, h / 6.0, 4.0 * h / 6.0, h / 6.0)
    mass[0, 0] = mass[-1, -1] = h / 3.0
    stiff = _tridiag(nn, -1.0 / h, 2.0 / h, -1.0 / h)
    stiff[0, 0] = stiff[-1, -1] = 1.0 / h
    e0 = np.zeros(nn)
    e0[0] = 1.0
    return Problem(
        n_u=nn, n_z=1, mass=mass, f=lambda u, z: -stiff @ u - z[0] * e0,
        f_u=lambda u, z: -stiff, f_z=lambda u, z: -e0.reshape(nn, 1),
        u0=np.cos(np.pi * h * np.arange(nn)), theta=theta, w_state=alpha1 * mass,
        w_control=np.array([[1.0]]), w_terminal=(alpha2 * mass) if alpha2 > 0.0 else None)


# --------------------------------------------------------------------------
# time discretisation (timedisc.py)
# --------------------------------------------------------------------------
def theta_residual(p: Problem, v, u, z, dt):
    """timedisc.py:112-130."""
    r = p.mass @ (v - u)
    if p.theta != 0.0:
        r = r + dt * p.theta * p.f(u, z)
    if p.theta != 1.0:
        r = r + dt * (1.0 - p.theta) * p.f(v, z)
    return r


def stage_jacobians(p: Problem, v, u, z, dt):
    """timedisc.py:133-149."""
    th = p.theta
    k = -p.mass + dt * th * p.f_u(u, z)
    c = p.mass + dt * (1.0 - th) * p.f_u(v, z)
    b = dt * th * p.f_z(u, z) + dt * (1.0 - th) * p.f_z(v, z)
    return k, c, b


def forward_solve(p: Problem, controls, n, dt, newton_tol=1e-12):
    """Newton-per-step theta-method march (timedisc.py:152-191)."""
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
                raise RuntimeError(f"Newton diverged at step {i + 1}")
        states[i] = u
        u_prev = u
    return states


@dataclass
class Stages:
    """StageBlocks (kkt.py:53-80)."""
    k: np.ndarray
    c: np.ndarray
    b: np.ndarray
    q_u: np.ndarray
    q_v: np.ndarray
    q_z: np.ndarray

    @property
    def n(self):
        return self.k.shape[0]


def build_stages(p: Problem, dt, u, v, z) -> Stages:
    """kkt.py:100-124 with stage_weights of timedisc.py:194-206."""
    n = u.shape[0]
    nu, nz = p.n_u, p.n_z
    k = np.empty((n, nu, nu)); c = np.empty((n, nu, nu)); b = np.empty((n, nu, nz))
    qu = np.empty((n, nu, nu)); qv = np.empty((n, nu, nu)); qz = np.empty((n, nz, nz))
    v_prev = np.asarray(p.u0, dtype=np.float64)
    for i in range(n):
        k[i], c[i], b[i] = stage_jacobians(p, v_prev, u[i], z[i], dt)
        q = 0.5 * dt * p.w_state
        if p.w_terminal is not None and i == n - 1:
            q = q + 0.5 * p.w_terminal
        qu[i], qv[i], qz[i] = q, q.copy(), dt * p.w_control
        v_prev = v[i]
    return Stages(k, c, b, qu, qv, qz)


# --------------------------------------------------------------------------
# the augmented operator (kkt.py)
# --------------------------------------------------------------------------
class Layout:
    """Time-clustered index map (kkt.py:127-191)."""

    def __init__(self, n, nu, nz):
        self.n, self.nu, self.nz = n, nu, nz
        self.first = 2 * nu + nz
        self.m = 4 * nu + nz
        self.last = 2 * nu
        self.dim = n * self.m
        starts = np.empty(n + 1, dtype=np.intp)
        starts[0] = 0
        starts[1:] = self.first + np.arange(n) * self.m
        self.starts = starts
        t = np.arange(1, n + 1)
        seg = lambda off, w: off[:, None] + np.arange(w)[None, :]
        self.rows = {
            "u": seg(np.where(t == 1, 0, starts[t - 1] + nu), nu),
            "z": seg(np.where(t == 1, nu, starts[t - 1] + 2 * nu), nz),
            "lam": seg(np.where(t == 1, nu + nz, starts[t - 1] + 3 * nu + nz), nu),
            "v": seg(starts[t], nu),
            "mu": seg(np.where(t == n, starts[t] + nu, starts[t] + 2 * nu + nz), nu),
        }

    def size(self, i):
        return self.first if i == 0 else (self.last if i == self.n else self.m)


class Kkt:
    """Figure-3 operator: diagonal blocks + identity continuity couplings
    (kkt.py:194-320)."""

    def __init__(self, s: Stages):
        n, nu, nz = s.n, s.k.shape[1], s.b.shape[2]
        self.n, self.nu, self.nz = n, nu, nz
        self.lay = Layout(n, nu, nz)
        eye = np.eye(nu)
        first = np.zeros((2 * nu + nz,) * 2)
        first[:nu, :nu] = s.q_u[0]
        first[nu:nu + nz, nu:nu + nz] = s.q_z[0]
        first[:nu, nu + nz:] = s.k[0].T
        first[nu:nu + nz, nu + nz:] = s.b[0].T
        first[nu + nz:, :nu] = s.k[0]
        first[nu + nz:, nu:nu + nz] = s.b[0]
        m = 4 * nu + nz
        inter = np.zeros((max(n - 1, 0), m, m))
        if n > 1:
            iv, iu, iz, imu, il = 0, nu, 2 * nu, 2 * nu + nz, 3 * nu + nz
            inter[:, iv:iv + nu, iv:iv + nu] = s.q_v[:-1]
            inter[:, iu:iu + nu, iu:iu + nu] = s.q_u[1:]
            inter[:, iz:iz + nz, iz:iz + nz] = s.q_z[1:]
            inter[:, iv:iv + nu, imu:imu + nu] = -eye
            inter[:, imu:imu + nu, iv:iv + nu] = -eye
            inter[:, iv:iv + nu, il:] = np.transpose(s.c[1:], (0, 2, 1))
            inter[:, iu:iu + nu, il:] = np.transpose(s.k[1:], (0, 2, 1))
            inter[:, iz:iz + nz, il:] = np.transpose(s.b[1:], (0, 2, 1))
            inter[:, il:, iv:iv + nu] = s.c[1:]
            inter[:, il:, iu:iu + nu] = s.k[1:]
            inter[:, il:, iz:iz + nz] = s.b[1:]
        last = np.zeros((2 * nu, 2 * nu))
        last[:nu, :nu] = s.q_v[-1]
        last[:nu, nu:] = -eye
        last[nu:, :nu] = -eye
        self.first, self.inter, self.last = first, inter, last

    @property
    def dim(self):
        return self.lay.dim

    def block(self, i):
        return self.first if i == 0 else (self.last if i == self.n else self.inter[i - 1])

    def apply_diag(self, x):
        lay = self.lay
        y = np.empty(lay.dim)
        f = lay.first
        y[:f] = self.first @ x[:f]
        if self.n > 1:
            m = lay.m
            y[f:f + (self.n - 1) * m] = np.matmul(
                self.inter, x[f:f + (self.n - 1) * m].reshape(self.n - 1, m, 1)).reshape(-1)
        y[-lay.last:] = self.last @ x[-lay.last:]
        return y

    def apply(self, x):
        """kkt.py:228-247."""
        y = self.apply_diag(x)
        mu, u = self.lay.rows["mu"], self.lay.rows["u"]
        y[mu] += x[u]
        y[u] += x[mu]
        return y

    def materialize(self):
        lay = self.lay
        a = np.zeros((lay.dim, lay.dim))
        for i in range(self.n + 1):
            s, w = lay.starts[i], lay.size(i)
            a[s:s + w, s:s + w] = self.block(i)
        mu, u = lay.rows["mu"].reshape(-1), lay.rows["u"].reshape(-1)
        a[mu, u] += 1.0
        a[u, mu] += 1.0
        return a


def _lu(a, floor=PIVOT_FLOOR):
    """linalg.py:76-99 (pivot-floor check)."""
    lu, piv = scipy.linalg.lu_factor(a, check_finite=False)
    n = a.shape[0]
    if n and np.abs(np.diag(lu)).min() < floor * max(float(np.abs(a).max()), 1e-300):
        raise np.linalg.LinAlgError("singular block")
    return lu, piv


class DiagSolve:
    """Explicit per-block inverses (kkt.py:338-389)."""

    def __init__(self, a: Kkt):
        self.a = a
        inv = lambda blk: scipy.linalg.lu_solve(_lu(blk), np.eye(blk.shape[0]),
                                                check_finite=False)
        self.inv_first = inv(a.first)
        self.inv_inter = np.array([inv(a.inter[i]) for i in range(a.n - 1)]) \
            if a.n > 1 else np.empty((0, 0, 0))
        self.inv_last = inv(a.last)

    def block(self, i, r):
        a = self.a
        if i == 0:
            return self.inv_first @ r
        if i == a.n:
            return self.inv_last @ r
        return self.inv_inter[i - 1] @ r

    def all(self, r):
        lay, a = self.a.lay, self.a
        out = np.empty(lay.dim)
        f = lay.first
        out[:f] = self.inv_first @ r[:f]
        if a.n > 1:
            m = lay.m
            out[f:f + (a.n - 1) * m] = np.matmul(
                self.inv_inter, r[f:f + (a.n - 1) * m].reshape(a.n - 1, m, 1)).reshape(-1)
        out[-lay.last:] = self.inv_last @ r[-lay.last:]
        return out


# --------------------------------------------------------------------------
# smoothers (smoothers.py)
# --------------------------------------------------------------------------
def jacobi(a: Kkt, d: DiagSolve, b, x, sweeps=1, omega=1.0):
    """smoothers.py:61-76."""
    x = np.array(x, dtype=np.float64)
    for _ in range(sweeps):
        x += omega * d.all(b - a.apply(x))
    return x


def _coupling_row(a: Kkt, i):
    """mu-row local offset of block i (kkt.py:221-226)."""
    return a.nu if i == a.n else 2 * a.nu + a.nz


def forward_subst(a: Kkt, d: DiagSolve, r):
    """(D - L) delta = r (smoothers.py:79-92)."""
    lay, nu = a.lay, a.nu
    delta = np.empty(lay.dim)
    for i in range(a.n + 1):
        s, w = lay.starts[i], lay.size(i)
        rhs = r[s:s + w].copy()
        if i >= 1:
            row = _coupling_row(a, i)
            rhs[row:row + nu] -= delta[lay.rows["u"][i - 1]]
        delta[s:s + w] = d.block(i, rhs)
    return delta


def backward_subst(a: Kkt, d: DiagSolve, r):
    """(D - U) delta = r (smoothers.py:95-109)."""
    lay, nu = a.lay, a.nu
    delta = np.empty(lay.dim)
    for i in range(a.n, -1, -1):
        s, w = lay.starts[i], lay.size(i)
        rhs = r[s:s + w].copy()
        if i <= a.n - 1:
            row = 0 if i == 0 else nu
            rhs[row:row + nu] -= delta[lay.rows["mu"][i]]
        delta[s:s + w] = d.block(i, rhs)
    return delta


def fgs(a, d, b, x):
    """smoothers.py:112-118."""
    return x + forward_subst(a, d, b - a.apply(x))


def bgs(a, d, b, x):
    """smoothers.py:121-127."""
    return x + backward_subst(a, d, b - a.apply(x))


def sgs(a, d, b, x):
    """P_sgs^{-1} r = (D-U)^{-1} D (D-L)^{-1} r (smoothers.py:130-152)."""
    r = b - a.apply(x)
    w = forward_subst(a, d, r)
    return x + backward_subst(a, d, a.apply_diag(w))


# --------------------------------------------------------------------------
# Krylov (krylov.py:77-210)
# --------------------------------------------------------------------------
@dataclass
class Report:
    iterations: int
    history: list
    converged: bool
    final_rel: float


def gmres_engine(op, prec, b, x0, rel_tol, max_iters, restart, flexible):
    """Right-preconditioned (F)GMRES, MGS Arnoldi + Givens (krylov.py:77-191)."""
    n = b.shape[0]
    x = np.zeros(n) if x0 is None else np.array(x0, dtype=np.float64)
    if restart is None:
        restart = max_iters
    r = b - op(x)
    beta0 = float(np.linalg.norm(r))
    hist = [beta0]
    if beta0 == 0.0:
        return x, Report(0, hist, True, 0.0)
    target = rel_tol * beta0
    total = 0
    while True:
        beta = float(np.linalg.norm(r))
        if beta <= target:
            break
        m = min(restart, max_iters - total)
        if m <= 0:
            break
        V = np.empty((m + 1, n))
        Z = np.empty((m, n)) if (flexible and prec is not None) else None
        H = np.zeros((m + 1, m)); cs = np.zeros(m); sn = np.zeros(m)
        g = np.zeros(m + 1); g[0] = beta
        V[0] = r / beta
        jd = 0
        broke = False
        for j in range(m):
            zj = V[j] if prec is None else prec(V[j])
            if Z is not None:
                Z[j] = zj
            w = op(zj)
            for i in range(j + 1):
                hij = float(np.dot(V[i], w))
                H[i, j] = hij
                w -= hij * V[i]
            hj1 = float(np.linalg.norm(w))
            H[j + 1, j] = hj1
            if not np.isfinite(hj1) or not np.isfinite(H[:j + 1, j]).all():
                raise FloatingPointError("non-finite Hessenberg entry")
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            den = float(np.hypot(H[j, j], H[j + 1, j]))
            if den == 0.0:
                raise FloatingPointError("Givens breakdown")
            cs[j] = H[j, j] / den
            sn[j] = H[j + 1, j] / den
            H[j, j] = den
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            total += 1
            jd = j + 1
            est = abs(g[j + 1])
            hist.append(est)
            if hj1 <= BREAKDOWN_TOL * beta0:
                broke = True
                break
            if est <= target or total >= max_iters:
                break
            V[j + 1] = w / hj1
        if jd > 0:
            y = np.zeros(jd)
            for i in range(jd - 1, -1, -1):
                y[i] = (g[i] - H[i, i + 1:jd] @ y[i + 1:jd]) / H[i, i]
            if Z is not None:
                x = x + Z[:jd].T @ y
            else:
                vy = V[:jd].T @ y
                x = x + (vy if prec is None else prec(vy))
        r = b - op(x)
        tn = float(np.linalg.norm(r))
        if broke and tn > max(target, 10 * BREAKDOWN_TOL * beta0):
            raise FloatingPointError("Arnoldi breakdown with nonzero residual")
        if tn <= target or total >= max_iters or broke:
            break
    fr = float(np.linalg.norm(b - op(x))) / beta0
    return x, Report(total, hist, fr <= rel_tol, fr)


def gmres(op, prec, b, x0=None, rel_tol=1e-10, max_iters=401, restart=None):
    return gmres_engine(op, prec, b, x0, rel_tol, max_iters, restart, False)


def fgmres(op, prec, b, x0=None, rel_tol=1e-10, max_iters=401, restart=None):
    return gmres_engine(op, prec, b, x0, rel_tol, max_iters, restart, True)


# --------------------------------------------------------------------------
# multigrid (multigrid.py)
# --------------------------------------------------------------------------
STATE_KINDS = ("u", "v", "lam", "mu")


def restrict_kkt(lf: Layout, lc: Layout, x):
    """multigrid.py:104-113: injection at even fine nodes, control average."""
    out = np.empty(lc.dim)
    for k in STATE_KINDS:
        out[lc.rows[k]] = x[lf.rows[k][1::2]]
    zf = lf.rows["z"]
    out[lc.rows["z"]] = 0.5 * (x[zf[0::2]] + x[zf[1::2]])
    return out


def prolong_kkt(lf: Layout, lc: Layout, x):
    """multigrid.py:115-132: linear interpolation / piecewise-constant copy."""
    out = np.empty(lf.dim)
    for k in STATE_KINDS:
        rc, rf = lc.rows[k], lf.rows[k]
        vals = x[rc]
        out[rf[1::2]] = vals
        out[rf[0]] = vals[0]
        if lc.n > 1:
            out[rf[2::2]] = 0.5 * (vals[:-1] + vals[1:])
    rc, rf = lc.rows["z"], lf.rows["z"]
    out[rf[0::2]] = x[rc]
    out[rf[1::2]] = x[rc]
    return out


@dataclass
class Level:
    n: int
    dt: float
    stages: Stages
    kkt: Kkt
    dsolve: DiagSolve


@dataclass
class Hierarchy:
    levels: List[Level]
    sweeps: int = 4
    omega: float = 1.0
    cycle_kind: str = "v"
    coarse_tol: float = 1e-2
    coarse_max_iters: int = 401
    coarse_calls: int = 0
    coarse_iters: int = 0


def default_levels(n_steps, coarsest=16):
    """multigrid.py:180-187."""
    levels, n = 1, n_steps
    while n % 2 == 0 and n // 2 >= coarsest:
        n //= 2
        levels += 1
    return levels


def build_hierarchy(p: Problem, u, v, z, n, dt, levels, sweeps=4, omega=1.0,
                    cycle_kind="v", coarse_tol=1e-2, coarse_max_iters=401):
    """Rediscretised ladder (multigrid.py:190-242)."""
    if n % (1 << (levels - 1)) != 0:
        raise ValueError("indivisible steps")
    lv = []
    u, v, z = (np.asarray(a, dtype=np.float64) for a in (u, v, z))
    nl, dtl = n, dt
    for ell in range(levels):
        st = build_stages(p, dtl, u, v, z)
        a = Kkt(st)
        lv.append(Level(nl, dtl, st, a, DiagSolve(a)))
        if ell < levels - 1:
            u, v = u[1::2], v[1::2]
            z = 0.5 * (z[0::2] + z[1::2])
            nl //= 2
            dtl *= 2.0
    return Hierarchy(lv, sweeps, omega, cycle_kind, coarse_tol, coarse_max_iters)


def coarse_solve(h: Hierarchy, r):
    """SGS-preconditioned GMRES from zero (multigrid.py:245-260)."""
    lev = h.levels[-1]
    zero = np.zeros(lev.kkt.dim)
    x, rep = gmres(lev.kkt.apply, lambda q: sgs(lev.kkt, lev.dsolve, q, zero), r,
                   None, h.coarse_tol, h.coarse_max_iters)
    h.coarse_calls += 1
    h.coarse_iters += rep.iterations
    return x


def cycle(h: Hierarchy, level, b, x0=None, kind=None):
    """Algorithm 1 generalised to V/F/W (multigrid.py:269-301)."""
    kind = h.cycle_kind if kind is None else kind
    lev = h.levels[level]
    if level == len(h.levels) - 1:
        return coarse_solve(h, b) if x0 is None else x0 + coarse_solve(h, b - lev.kkt.apply(x0))
    x = np.zeros(lev.kkt.dim) if x0 is None else np.asarray(x0, dtype=np.float64)
    x = jacobi(lev.kkt, lev.dsolve, b, x, h.sweeps, h.omega)
    lf, lc = lev.kkt.lay, h.levels[level + 1].kkt.lay
    r = restrict_kkt(lf, lc, b - lev.kkt.apply(x))
    if kind == "v":
        e = cycle(h, level + 1, r, None, "v")
    elif kind == "w":
        e = cycle(h, level + 1, r, None, "w")
        e = cycle(h, level + 1, r, e, "w")
    else:
        e = cycle(h, level + 1, r, None, "f")
        e = cycle(h, level + 1, r, e, "v")
    x = x + prolong_kkt(lf, lc, e)
    return jacobi(lev.kkt, lev.dsolve, b, x, h.sweeps, h.omega)


def mg_prec(h: Hierarchy):
    """multigrid.py:304-311."""
    return lambda r: cycle(h, 0, r)
