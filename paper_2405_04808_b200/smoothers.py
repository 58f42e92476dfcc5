"""Fixed-point operators over A = D - L - U (reference smoothers.py):
block Jacobi (one fused residual+local-solve kernel per sweep, parallel over
time intervals) and forward / backward / symmetric block Gauss-Seidel
(serial-in-time substitution kernels).  Device tensors in/out; numpy in ->
numpy out.
"""

from __future__ import annotations

from . import device as dev
from .errors import DimensionMismatch
from .kkt import FAMILY_TRI, BlockTriKKT, DiagonalSolver
from .krylov import Preconditioner

SMOOTHER_KINDS = ("jacobi", "fgs", "bgs", "sgs")


def _prep(a: BlockTriKKT, b, x):
    host = dev.is_host(b)
    b = dev.to_device(b)
    x = None if x is None else dev.to_device(x)
    if b.shape != (a.dim,) or (x is not None and x.shape != (a.dim,)):
        raise DimensionMismatch("vector length does not match the operator")
    return host, b, x


def jacobi_sweeps(a: BlockTriKKT, b, x, sweeps: int = 1, omega: float = 1.0, out=None):
    """x <- x + omega*D^{-1}(b - A x), `sweeps` times, on device tensors.
    ``x`` may be None (zero initial guess: the first sweep is D^{-1} b)."""
    cur = x
    buf = [dev.empty(a.dim) if out is None else out, None]
    for k in range(sweeps):
        dst = buf[k & 1]
        if dst is None or dst is cur:
            dst = buf[k & 1] = dev.empty(a.dim)
        dev.call("tk_jacobi_sweep", a.lref, dev.P(b), dev.P(cur), dev.P(dst), omega,
                 dev.stream())
        cur = dst
    return cur


def jacobi_apply(a: BlockTriKKT, dfac, b, x, sweeps: int = 1, omega: float = 1.0):
    """Block-Jacobi relaxation (smoothers.py:61-76)."""
    host, b, x = _prep(a, b, x)
    out = jacobi_sweeps(a, b, x, sweeps, omega)
    return dev.to_host(out) if host else out


def forward_subst(a: BlockTriKKT, r, out=None):
    """Solve (D - L) delta = r (smoothers.py:79-92)."""
    a.ensure_subst()
    d = dev.empty(a.dim) if out is None else out
    dev.call("tk_forward_subst", a.lref, dev.P(r), dev.P(d), dev.stream())
    return d


def backward_subst(a: BlockTriKKT, r, out=None):
    """Solve (D - U) delta = r (smoothers.py:95-109)."""
    a.ensure_subst()
    d = dev.empty(a.dim) if out is None else out
    dev.call("tk_backward_subst", a.lref, dev.P(r), dev.P(d), dev.stream())
    return d


def _residual(a, b, x):
    return b.clone() if x is None else a.residual(b, x)


def fgs_apply(a: BlockTriKKT, dfac, b, x):
    """x + (D - L)^{-1}(b - A x) (smoothers.py:112-118)."""
    host, b, x = _prep(a, b, x)
    d = forward_subst(a, _residual(a, b, x))
    if x is not None:
        d += x
    return dev.to_host(d) if host else d


def bgs_apply(a: BlockTriKKT, dfac, b, x):
    """x + (D - U)^{-1}(b - A x) (smoothers.py:121-127)."""
    host, b, x = _prep(a, b, x)
    d = backward_subst(a, _residual(a, b, x))
    if x is not None:
        d += x
    return dev.to_host(d) if host else d


def sgs_zero(a: BlockTriKKT, r, out=None):
    """P_sgs^{-1} r = (D-U)^{-1} D (D-L)^{-1} r, i.e. sgs_apply from x = 0.
    TRI levels with factor records fuse `D` and the backward substitution's
    D^{-1} (tk_sgs_back_half: the backward chain starts from w itself)."""
    w = forward_subst(a, r)
    if a.family == FAMILY_TRI and a.has_records and not a.is_slab:
        d = dev.empty(a.dim) if out is None else out
        dev.call("tk_sgs_back_half", a.lref, dev.P(w), dev.P(d), dev.stream())
        return d
    y = a.apply_diag(w)
    return backward_subst(a, y, out=out)


def sgs_apply(a: BlockTriKKT, dfac, b, x):
    """Symmetric block Gauss-Seidel update (smoothers.py:130-152)."""
    host, b, x = _prep(a, b, x)
    d = sgs_zero(a, _residual(a, b, x))
    if x is not None:
        d += x
    return dev.to_host(d) if host else d


def smoother_preconditioner(a: BlockTriKKT, dfac, kind: str, sweeps: int = 1,
                            omega: float = 1.0) -> Preconditioner:
    """One fixed-point application from zero as a right preconditioner
    (smoothers.py:155-168); a fixed linear map, hence not flexible."""
    if kind not in SMOOTHER_KINDS:
        raise ValueError(f"unknown smoother kind {kind!r}")
    if kind == "jacobi":
        return Preconditioner(apply=lambda r: jacobi_apply(a, dfac, r, None, sweeps, omega),
                              is_flexible=False)
    if kind == "sgs":
        return Preconditioner(apply=lambda r: _host_wrap(sgs_zero, a, r), is_flexible=False)
    fn = forward_subst if kind == "fgs" else backward_subst
    return Preconditioner(apply=lambda r: _host_wrap(fn, a, r), is_flexible=False)


def _host_wrap(fn, a, r):
    host = dev.is_host(r)
    out = fn(a, dev.to_device(r))
    return dev.to_host(out) if host else out
