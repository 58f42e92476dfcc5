"""Right-preconditioned (F)GMRES with device-resident Krylov bases
(reference krylov.py:77-210).

Same algorithm, stopping rules and reports as the reference -- modified
Gram-Schmidt Arnoldi, Givens rotations, restarts, happy-breakdown test --
so iteration counts and residual histories match it.  The basis V (and Z
for FGMRES) live in HBM; every vector operation is a libtempokkt_b200.so
kernel (deterministic reductions) and only the Hessenberg scalars come back
to the host.  numpy right-hand sides are accepted (the solution is returned
as numpy).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import Callable

import os

import numpy as np
import torch

from . import _lib
from . import device as dev
from .errors import Breakdown, DimensionMismatch, NonFiniteValue

BREAKDOWN_TOL = 1e-14
# MGS Arnoldi step as one cooperative launch (tk_arnoldi_mgs) instead of
# j+1 dot/axpy pairs with a host round trip each; bitwise identical
FUSED_ARNOLDI = True
# Krylov bases above this size are allocated at their full length at once
GROW_LIMIT_BYTES = 2 << 30


@dataclass
class LinearOperator:
    dim: int
    apply: Callable

    def __call__(self, x):
        return self.apply(x)


@dataclass
class Preconditioner:
    apply: Callable
    is_flexible: bool = False

    def __call__(self, r):
        return self.apply(r)


@dataclass
class SolveReport:
    iterations: int
    residual_history: list = field(default_factory=list)
    converged: bool = False
    final_relative_residual: float = float("nan")


class MappedScalars:
    """Pinned host memory mapped into the device address space
    (tk_host_alloc_mapped).  Reduction kernels write their scalars straight
    into it and the host reads them after a stream synchronisation; uploads
    go through tk_copy_kernel.  No scalar crosses PCIe on a copy engine, so
    the Krylov recurrence never queues behind a bulk host<->device copy of
    another stream (HostPipeline)."""

    def __init__(self, n: int):
        lib = _lib.load()
        h, d = ctypes.c_void_p(), ctypes.c_void_p()
        _lib.check(lib.tk_host_alloc_mapped(8 * n, ctypes.byref(h), ctypes.byref(d)),
                   "tk_host_alloc_mapped")
        self.n = n
        self.host_ptr, self.dev_ptr = h.value, d.value
        self.host = np.ctypeslib.as_array((ctypes.c_double * n).from_address(h.value))

    def dptr(self, k: int = 0) -> int:
        return self.dev_ptr + 8 * k

    def __del__(self):
        try:
            _lib.load().tk_host_free(ctypes.c_void_p(self.host_ptr))
        except Exception:
            pass


def _sync():
    torch.cuda.current_stream().synchronize()


class VecOps:
    """Thin wrapper over the BLAS-1 kernels; scalars live in mapped pinned
    memory (MappedScalars)."""

    def __init__(self):
        lib = _lib.load()
        self.work = dev.empty(int(lib.tk_reduce_work_len()))
        self.scal = dev.empty(8)
        self.ms = MappedScalars(8)
        self.hmap = None        # Hessenberg column (grown on demand)
        self.cdev = None        # uploaded gemv coefficients
        self.cmap = None

    def dot_dev(self, x, y, slot=0):
        """<x, y> into the device scalar self.scal[slot] (no host sync)."""
        dev.call("tk_dot", x.numel(), dev.P(x), dev.P(y), self.scal[slot:].data_ptr(),
                 dev.P(self.work), dev.stream())
        return self.scal[slot]

    def dot(self, x, y) -> float:
        dev.call("tk_dot", x.numel(), dev.P(x), dev.P(y), self.ms.dptr(0), dev.P(self.work),
                 dev.stream())
        _sync()
        return float(self.ms.host[0])

    def nrm2(self, x) -> float:
        dev.call("tk_nrm2", x.numel(), dev.P(x), self.ms.dptr(1), dev.P(self.work),
                 dev.stream())
        _sync()
        return float(self.ms.host[1])

    def nrm2_async(self, x, slot: int):
        """||x|| into mapped slot `slot` (2..7); read it after the next sync."""
        dev.call("tk_nrm2", x.numel(), dev.P(x), self.ms.dptr(slot), dev.P(self.work),
                 dev.stream())

    def axpy(self, a, x, y):
        dev.call("tk_axpy", x.numel(), float(a), dev.P(x), dev.P(y), dev.stream())

    def scale_into(self, a, x, y):
        dev.call("tk_scale_into", x.numel(), float(a), dev.P(x), dev.P(y), dev.stream())

    def arnoldi(self, V, j, w):
        """MGS step against V[0..j] in one launch (tk_arnoldi_mgs): returns
        h_0..h_{j+1} (written by the kernel into mapped host memory); w is
        orthogonalised in place and V[j+1] = w / h_{j+1}."""
        k = j + 2
        if self.hmap is None or self.hmap.n < k:
            self.hmap = MappedScalars(max(k, 2 * (self.hmap.n if self.hmap else 64)))
        dev.call("tk_arnoldi_mgs", w.numel(), j, dev.P(V), V.stride(0), dev.P(w),
                 self.hmap.dptr(), dev.P(self.work), dev.stream())
        _sync()
        return self.hmap.host[:k].copy()

    def gemv_t_add(self, V, c, x):
        """x += V[:k]^T c (V rows contiguous; c numpy or torch)."""
        k = int(c.numel()) if isinstance(c, torch.Tensor) else int(np.size(c))
        if k == 0:
            return
        if isinstance(c, torch.Tensor) and c.is_cuda:
            cd = c.contiguous()
        else:
            if self.cmap is None or self.cmap.n < k:
                self.cmap = MappedScalars(max(k, 2 * (self.cmap.n if self.cmap else 64)))
                self.cdev = dev.empty(self.cmap.n)
            _sync()                      # the previous upload has been consumed
            self.cmap.host[:k] = np.asarray(c.cpu() if isinstance(c, torch.Tensor) else c,
                                            dtype=np.float64)
            dev.call("tk_copy_kernel", k, self.cmap.dptr(), dev.P(self.cdev), dev.stream())
            cd = self.cdev
        dev.call("tk_gemv_t_add", x.numel(), k, dev.P(V), V.stride(0), dev.P(cd), dev.P(x),
                 dev.stream())


_OPS = None
_FUSED_OK = {}


def fused_arnoldi_ok() -> bool:
    """The cooperative Arnoldi grid fits the current device (else the unfused
    kernels run: same reductions, same bits)."""
    d = torch.cuda.current_device()
    if d not in _FUSED_OK:
        _FUSED_OK[d] = bool(_lib.load().tk_arnoldi_supported())
    return _FUSED_OK[d]


def vec_ops() -> VecOps:
    global _OPS
    if _OPS is None:
        _OPS = VecOps()
    return _OPS


def _as_prec(prec):
    if prec is None or isinstance(prec, Preconditioner):
        return prec
    return Preconditioner(apply=prec)


def _residual(op, b, x):
    """r = b - op(x) with the rsub kernel (op(x) is a fresh tensor)."""
    y = dev.to_device(op(x))
    dev.call("tk_rsub", y.numel(), dev.P(b), dev.P(y), dev.stream())
    return y


class DeviceSpace:
    """The vector space of a single-GPU solve: every operation a
    libtempokkt_b200.so kernel on whole vectors (VecOps)."""

    def __init__(self):
        self.ops = vec_ops()

    def nrm2(self, x) -> float:
        return self.ops.nrm2(x)

    def nrm2_pair(self, x, r):
        """(||x||, ||r||) with one synchronisation."""
        self.ops.nrm2_async(x, 2)        # the finiteness check rides on the next sync
        rn = self.ops.nrm2(r)
        return float(self.ops.ms.host[2]), rn

    def scale_into(self, a, x, y):
        self.ops.scale_into(a, x, y)

    def axpy(self, a, x, y):
        self.ops.axpy(a, x, y)

    def arnoldi(self, V, j, w):
        if FUSED_ARNOLDI and fused_arnoldi_ok():   # one launch + one copy per step
            return self.ops.arnoldi(V, j, w)
        hcol = np.empty(j + 2)
        for i in range(j + 1):
            hij = self.ops.dot(V[i], w)
            hcol[i] = hij
            self.ops.axpy(-hij, V[i], w)
        hcol[j + 1] = self.ops.nrm2(w)
        if hcol[j + 1] != 0.0:
            self.ops.scale_into(1.0 / hcol[j + 1], w, V[j + 1])
        return hcol

    def gemv_t_add(self, V, c, x):
        self.ops.gemv_t_add(V, c, x)

    def residual(self, op, b, x):
        return _residual(op, b, x)

    def finish(self):
        # the Arnoldi steps of a large basis held w L2-persisting (tk_arnoldi_mgs):
        # give the lines back once the solve has synchronised
        _lib.check(_lib.load().tk_l2_persist_reset(), "tk_l2_persist_reset")


_DEPTH = [0]          # nesting of solves (the coarse GMRES runs inside the outer one)


def _gmres_engine(op, prec, b, x0, rel_tol, max_iters, restart, flexible, space=None):
    """Right-preconditioned (F)GMRES with restarts (krylov.py:77-191): same
    modified Gram-Schmidt Arnoldi, Givens rotations, stopping and breakdown
    rules and reports as the reference.  ``space`` supplies the vector
    operations (DeviceSpace: one GPU; slabs.SlabSpace: time slabs over ranks
    with allreduced dots)."""
    space = DeviceSpace() if space is None else space
    lib = _lib.load()
    _DEPTH[0] += 1
    lib.tk_l2_persist_allow(1 if _DEPTH[0] == 1 else 0)   # only the outermost solve's w persists
    try:
        return _gmres_body(op, prec, b, x0, rel_tol, max_iters, restart, flexible, space)
    finally:
        _DEPTH[0] -= 1
        if _DEPTH[0] == 0:          # outermost solve only (also on an exception)
            space.finish()
        lib.tk_l2_persist_allow(1 if _DEPTH[0] <= 1 else 0)


def _gmres_body(op, prec, b, x0, rel_tol, max_iters, restart, flexible, space):
    if not (0.0 < rel_tol < 1.0):
        raise ValueError(f"rel_tol must lie in (0,1), got {rel_tol}")
    n = op.dim
    host = dev.is_host(b)
    b = dev.to_device(b) if not hasattr(space, "to_local") else space.to_local(b)
    if b.shape != (n,):
        raise DimensionMismatch(f"rhs shape {tuple(b.shape)} != operator dim {n}")
    prec = _as_prec(prec)
    if restart is None:
        restart = max_iters
    if restart < 1:
        raise ValueError("restart must be >= 1")
    if x0 is None:
        r = b.clone()                      # b - A*0, bitwise
        x = torch.empty_like(b)
        space.scale_into(0.0, r, x)        # x = 0 (signed zeros add exactly)
    else:
        x = (dev.to_device(x0) if not hasattr(space, "to_local") else space.to_local(x0)).clone()
        if x.shape != (n,):
            raise DimensionMismatch(f"x0 shape {tuple(x.shape)} != operator dim {n}")
        r = space.residual(op, b, x)
    beta0 = space.nrm2(r)
    if not math.isfinite(beta0):
        raise NonFiniteValue("non-finite initial residual")
    history = [beta0]
    if beta0 == 0.0:
        rep = SolveReport(0, history, True, 0.0)
        return (dev.to_host(x) if host else x), rep
    target = rel_tol * beta0
    x_norm = true_norm = None
    total = 0
    beta = beta0
    while True:
        if beta <= target:
            break
        m = min(restart, max_iters - total)
        if m <= 0:
            break
        # bases grow on demand (doubling): a coarse solve that stops after a
        # few iterations does not hold max_iters+1 vectors of HBM; bases whose
        # full size exceeds GROW_LIMIT_BYTES (outer solves of the large
        # configurations, restart sized to the free HBM) are allocated once,
        # since growing would hold the old and the new basis side by side
        nb = 2 if (flexible and prec is not None) else 1
        cap = m if (m + 1) * n * 8 * nb > GROW_LIMIT_BYTES else min(m, 16)
        V = torch.empty((cap + 1, n), dtype=b.dtype, device=b.device)
        Z = torch.empty((cap, n), dtype=b.dtype, device=b.device) \
            if (flexible and prec is not None) else None
        H = np.zeros((m + 1, m)); cs = [0.0] * m; sn = [0.0] * m
        g = [0.0] * (m + 1)
        g[0] = beta
        space.scale_into(1.0 / beta, r, V[0])
        jd = 0
        broke = False
        for j in range(m):
            if j + 1 > cap:
                cap = min(m, 2 * cap)
                V2 = torch.empty((cap + 1, n), dtype=b.dtype, device=b.device)
                V2[:j + 1].copy_(V[:j + 1])
                V = V2
                if Z is not None:
                    Z2 = torch.empty((cap, n), dtype=b.dtype, device=b.device)
                    Z2[:j].copy_(Z[:j])
                    Z = Z2
                V2 = Z2 = None
            if prec is None:
                zj = V[j]
            else:
                zj = prec(V[j])
                if Z is not None:
                    Z[j].copy_(zj)
                    zj = Z[j]
            w = op(zj)
            w = dev.to_device(w) if not hasattr(space, "to_local") else space.to_local(w)
            hcol = space.arnoldi(V, j, w)       # MGS; V[j+1] = w / h_{j+1} written too
            hj1 = float(hcol[j + 1])
            if not np.isfinite(hcol).all():
                raise NonFiniteValue("non-finite Hessenberg entry in Arnoldi")
            # Givens rotations on the new column as Python floats (same IEEE
            # arithmetic as numpy scalars, without per-element array access)
            col = hcol.tolist()
            for i in range(j):
                a_, b_ = col[i], col[i + 1]
                col[i] = cs[i] * a_ + sn[i] * b_
                col[i + 1] = -sn[i] * a_ + cs[i] * b_
            den = float(np.hypot(col[j], col[j + 1]))
            if den == 0.0:
                raise Breakdown("zero diagonal in Givens elimination")
            cs[j] = col[j] / den
            sn[j] = col[j + 1] / den
            col[j] = den
            col[j + 1] = 0.0
            H[:j + 2, j] = col
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            total += 1
            jd = j + 1
            est = abs(g[j + 1])
            history.append(est)
            if hj1 <= BREAKDOWN_TOL * beta0:
                broke = True
                break
            if est <= target or total >= max_iters:
                break
        if jd > 0:
            y = np.zeros(jd)
            for i in range(jd - 1, -1, -1):
                y[i] = (np.float64(g[i]) - H[i, i + 1:jd] @ y[i + 1:jd]) / H[i, i]
            yt = y
            if Z is not None:
                space.gemv_t_add(Z, yt, x)
            else:
                vy = torch.empty_like(b)
                space.scale_into(0.0, V[0], vy)
                space.gemv_t_add(V, yt, vy)
                if prec is not None:
                    pv = prec(vy)
                    vy = dev.to_device(pv) if not hasattr(space, "to_local") else \
                        space.to_local(pv)
                space.axpy(1.0, vy, x)
        zj = w = None        # views of Z / V: drop them so the bases are freed before a restart
        del V, Z
        r = space.residual(op, b, x)
        x_norm, true_norm = space.nrm2_pair(x, r)
        beta = true_norm
        if broke and true_norm > max(target, 10 * BREAKDOWN_TOL * beta0):
            raise Breakdown("zero Arnoldi norm with nonzero residual")
        if true_norm <= target or total >= max_iters or broke:
            break
    if x_norm is None:                    # no cycle ran (max_iters == 0)
        x_norm = space.nrm2(x)
        true_norm = space.nrm2(space.residual(op, b, x))
    if not math.isfinite(x_norm):
        raise NonFiniteValue("non-finite solution vector")
    # ||b - A x|| of the final x: the deterministic kernels give the bits the
    # loop's last true residual already has, so it is reused
    final_rel = true_norm / beta0
    report = SolveReport(iterations=total, residual_history=history,
                         converged=final_rel <= rel_tol, final_relative_residual=final_rel)
    return (dev.to_host(x) if host else x), report


def gmres(op, prec, b, x0=None, rel_tol=1e-10, max_iters=401, restart=None):
    """Restarted right-preconditioned GMRES (krylov.py:194-201)."""
    return _gmres_engine(op, prec, b, x0, rel_tol, max_iters, restart, flexible=False)


def fgmres(op, prec, b, x0=None, rel_tol=1e-10, max_iters=401, restart=None):
    """Flexible GMRES (krylov.py:204-210)."""
    return _gmres_engine(op, prec, b, x0, rel_tol, max_iters, restart, flexible=True)
