"""A V-cycle replayed as one CUDA graph (reference multigrid.py:269-301 with
the coarse solve of multigrid.py:245-260).

The eager cycle (multigrid._cycle) is host-driven: the coarse SGS-GMRES
synchronises with the host after its initial norm, after every Arnoldi step
(Givens update + stopping test), for the coefficient upload and for the
true-residual check, and the GPU idles while Python issues the next
launches.  ``VCycleGraph`` records levels 1..L-1 of one V-cycle once into a
CUDA graph in which the coarse GMRES is a device-side WHILE loop
(csrc/tk_graph.cu: the Givens kernel sets the loop condition), so a cycle is

    fine pre-smoothing + restricted residual   (two launches, any input b)
    -> ONE graph launch (all coarser levels, coarse solve included)
    -> prolongation + fine post-smoothing      (two launches)
    -> one synchronisation to read (fallback flag, coarse iterations).

The kernels and their order are the eager path's, so the result equals the
eager cycle's (the coarse scalar recurrence rounds like the host's; hypot
and the back-substitution's summation may differ in the last bit).  When
the device solve flags a case the host path handles differently (a restart,
breakdown, a non-finite value, more than ``cap`` coarse iterations) the
cycle is re-run eagerly, which reproduces the reference's behaviour,
exceptions included.  All buffers are allocated before capture; nothing is
allocated while capturing.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import _lib
from . import device as dev
from .kkt import FAMILY_TRI

# environment switch: TK_GRAPH=0 keeps every cycle eager
ENABLED = os.environ.get("TK_GRAPH", "1") != "0"
# the device coarse GMRES keeps z_j = M^{-1} v_j and forms x = Z y: one SGS
# application fewer per coarse solve than M^{-1}(V y) (the same vector for the
# fixed linear SGS preconditioner); TK_COARSE_ZBASIS=0 keeps the reference form
ZBASIS = os.environ.get("TK_COARSE_ZBASIS", "1") != "0"
DEFAULT_CAP = 64


class MappedInts:
    """Two int32 in mapped pinned host memory (written by gm_finish)."""

    def __init__(self):
        lib = _lib.load()
        h, d = ctypes.c_void_p(), ctypes.c_void_p()
        _lib.check(lib.tk_host_alloc_mapped(64, ctypes.byref(h), ctypes.byref(d)),
                   "tk_host_alloc_mapped")
        self.host_ptr, self.dev_ptr = h.value, d.value
        self.host = np.ctypeslib.as_array((ctypes.c_int32 * 16).from_address(h.value))

    def __del__(self):
        try:
            _lib.load().tk_host_free(ctypes.c_void_p(self.host_ptr))
        except Exception:
            pass


def supported(h) -> bool:
    """Graph replay covers single-GPU V-cycles with at least two levels."""
    if not ENABLED or h.n_levels < 2 or h.cycle_kind != "v":
        return False
    from .krylov import fused_arnoldi_ok
    if not fused_arnoldi_ok():         # the device GMRES uses the cooperative Arnoldi step
        return False
    return not any(lv.kkt.is_slab for lv in h.levels)


class VCycleGraph:
    """Levels 1..L-1 of a V-cycle from zero, captured once (see module doc)."""

    def __init__(self, h, cap: int = DEFAULT_CAP, start: int = 1):
        """start = 1: levels 1..L-1 of a V-cycle; start = L-1: the coarse
        solve alone (used for the coarse level gathered on one GPU)."""
        self.h = h
        self.start = start
        self.key = (h.sweeps, float(h.omega), float(h.coarse_tol), int(h.coarse_max_iters))
        self.cap = max(1, min(int(cap), int(h.coarse_max_iters)))
        lib = _lib.load()
        L = h.n_levels
        self.B = [None] * L          # level rhs (B[1] is the graph input)
        self.X = [None] * L          # pre-smoothed iterate
        self.Y = [None] * L          # second sweep buffer (sweeps > 1)
        self.E = [None] * L          # level correction (E[1] is the graph output)
        self.W = [None] * L          # residual work (general residual-restrict)
        for l in range(start, L):
            n = h.levels[l].kkt.dim
            self.B[l] = dev.empty(n)
            self.E[l] = dev.empty(n)
            if l < L - 1:
                self.X[l] = dev.empty(n)
                if h.sweeps > 1:
                    self.Y[l] = dev.empty(n)
                    self.W[l] = dev.empty(n)
        ac = h.levels[-1].kkt
        nc = ac.dim
        self.nc = nc
        self.V = dev.empty(self.cap + 1, nc)
        self.Z = dev.empty(self.cap, nc) if ZBASIS else None
        self.vj, self.zj, self.w, self.w1, self.vy, self.r = (dev.empty(nc) for _ in range(6))
        self.w2 = dev.empty(nc) if not self._fused_back_half(ac) else None
        self.state = dev.empty(int(lib.tk_gm_state_len(self.cap)))
        nw = int(lib.tk_reduce_work_len())
        self.work = dev.empty(nw)
        self.res = MappedInts()
        self.exec = None
        self._capture()

    @staticmethod
    def _fused_back_half(a) -> bool:
        return a.family == FAMILY_TRI and a.has_records and not a.is_slab

    # --- recording --------------------------------------------------------
    def _sgs(self, a, r, out):
        """P_sgs^{-1} r into out (smoothers.sgs_zero with fixed buffers)."""
        s = dev.stream()
        dev.call("tk_forward_subst", a.lref, dev.P(r), dev.P(self.w1), s)
        if self._fused_back_half(a):
            dev.call("tk_sgs_back_half", a.lref, dev.P(self.w1), dev.P(out), s)
        else:
            dev.call("tk_kkt_apply_diag", a.lref, dev.P(self.w1), dev.P(self.w2), s)
            dev.call("tk_backward_subst", a.lref, dev.P(self.w2), dev.P(out), s)

    def _sweeps(self, a, b, x, bufs, n_sweeps):
        """n_sweeps Jacobi sweeps from x (None: zero); the last lands in bufs[-1]."""
        cur = x
        seq = [bufs[(n_sweeps - 1 - k) % len(bufs)] for k in range(n_sweeps)]
        for k in range(n_sweeps):
            dst = seq[k]
            if dst is cur:
                raise RuntimeError("graph sweep buffers alias")
            dev.call("tk_jacobi_sweep", a.lref, dev.P(b), dev.P(cur), dev.P(dst),
                     float(self.h.omega), dev.stream())
            cur = dst
        return cur

    def _record_level(self, l, body_stream):
        from .multigrid import JACOBI0_RESIDUAL, fused_jacobi0_ok, fused_v11_ok, fused_vnn_ok
        h = self.h
        L = h.n_levels
        a = h.levels[l].kkt
        s = dev.stream()
        if l == L - 1:
            self._record_coarse(a, self.B[l], self.E[l], body_stream)
            return
        if fused_v11_ok(h, a) and fused_jacobi0_ok(a, h.omega):
            # V(1,1), omega = 1: pre-smoothing storing u / mu only, prolongation
            # inside the post-smoothing sweep
            dev.call("tk_jacobi0_restrict_um", a.lref, dev.P(self.B[l]), dev.P(self.X[l]),
                     dev.P(self.B[l + 1]), s)
            self._record_level(l + 1, body_stream)
            dev.call("tk_jacobi_prolong", a.lref, dev.P(self.B[l]), dev.P(self.X[l]),
                     dev.P(self.E[l + 1]), dev.P(self.E[l]), s)
            return
        if h.sweeps > 1 and fused_vnn_ok(h, a):
            # omega = 1, several sweeps: the last pre-smoothing sweep writes the
            # restricted residual, the first post-smoothing sweep prolongs
            xi = self._sweeps(a, self.B[l], None, [self.W[l], self.Y[l]], h.sweeps - 1)
            dev.call("tk_jacobi_restrict", a.lref, dev.P(self.B[l]), dev.P(xi), dev.P(self.X[l]),
                     dev.P(self.B[l + 1]), s)
            self._record_level(l + 1, body_stream)
            dev.call("tk_jacobi_prolong", a.lref, dev.P(self.B[l]), dev.P(self.X[l]),
                     dev.P(self.E[l + 1]), dev.P(self.Y[l]), s)
            self._sweeps(a, self.B[l], self.Y[l], [self.E[l], self.W[l]], h.sweeps - 1)
            return
        # pre-smoothing from zero: X (sweeps 1) or X/Y ping-pong ending in X
        bufs = [self.X[l]] if h.sweeps == 1 else [self.X[l], self.Y[l]]
        if h.sweeps == 1 and JACOBI0_RESIDUAL and fused_jacobi0_ok(a, h.omega):
            x = self.X[l]
            dev.call("tk_jacobi0_restrict", a.lref, dev.P(self.B[l]), float(h.omega), dev.P(x),
                     dev.P(self.B[l + 1]), s)
        else:
            x = self._sweeps(a, self.B[l], None, bufs, h.sweeps)
        if h.sweeps == 1 and JACOBI0_RESIDUAL and fused_jacobi0_ok(a, h.omega):
            pass
        elif h.sweeps == 1 and JACOBI0_RESIDUAL:
            dev.call("tk_residual_restrict_jacobi0", a.lref, dev.P(self.B[l]), dev.P(x),
                     float(h.omega), dev.P(self.B[l + 1]), s)
        else:
            dev.call("tk_residual_restrict", a.lref, dev.P(self.B[l]), dev.P(x),
                     dev.P(self.B[l + 1]), dev.P(self.W[l]), s)
        self._record_level(l + 1, body_stream)
        h.transfers[l].prolong_add(self.E[l + 1], x)
        other = [b for b in (self.X[l], self.Y[l]) if b is not None and b is not x]
        bufs = [self.E[l]] if h.sweeps == 1 else [self.E[l], other[0] if other else self.W[l]]
        self._sweeps(a, self.B[l], x, bufs, h.sweeps)

    def _record_coarse(self, a, b, x, body_stream):
        lib = _lib.load()
        h = self.h
        s = dev.stream()
        nc, cap, ld = self.nc, self.cap, self.V.stride(0)
        handle = ctypes.c_uint64()
        _lib.check(lib.tk_graph_cond_create(s, ctypes.byref(handle)), "tk_graph_cond_create")
        dev.call("tk_gm_begin", nc, dev.P(b), dev.P(self.V), ld, dev.P(self.vj),
                 dev.P(self.state), cap, float(h.coarse_tol), int(h.coarse_max_iters),
                 handle.value, dev.P(self.work), s)
        _lib.check(lib.tk_graph_while_begin(s, body_stream.cuda_stream, handle.value),
                   "tk_graph_while_begin")
        with torch.cuda.stream(body_stream):
            bs = dev.stream()
            self._sgs(a, self.vj, self.zj)
            if self.Z is not None:
                dev.call("tk_gm_storez", nc, dev.P(self.zj), dev.P(self.Z), self.Z.stride(0),
                         dev.P(self.state), cap, bs)
            dev.call("tk_kkt_apply", a.lref, dev.P(self.zj), dev.P(self.w), bs)
            dev.call("tk_gm_arnoldi", nc, dev.P(self.V), ld, dev.P(self.w), dev.P(self.state),
                     cap, dev.P(self.vj), dev.P(self.work), bs)
            dev.call("tk_gm_givens", dev.P(self.state), cap, handle.value, bs)
        _lib.check(lib.tk_graph_while_end(body_stream.cuda_stream), "tk_graph_while_end")
        if self.Z is not None:       # x = Z y
            dev.call("tk_gm_combine", nc, dev.P(self.Z), self.Z.stride(0), dev.P(self.state), cap,
                     dev.P(x), s)
        else:                        # x = M^{-1} (V y)
            dev.call("tk_gm_combine", nc, dev.P(self.V), ld, dev.P(self.state), cap,
                     dev.P(self.vy), s)
            self._sgs(a, self.vy, x)
        dev.call("tk_kkt_apply", a.lref, dev.P(x), dev.P(self.r), s)
        dev.call("tk_gm_finish", nc, dev.P(b), dev.P(self.r), dev.P(x), dev.P(self.state), cap,
                 self.res.dev_ptr, dev.P(self.work), s)

    def _capture(self):
        lib = _lib.load()
        cap_stream = torch.cuda.Stream()
        body_stream = torch.cuda.Stream()
        torch.cuda.synchronize()
        counting = dev.INSTR.counting
        dev.INSTR.counting = False
        ex = ctypes.c_void_p()
        with torch.cuda.stream(cap_stream):
            s = dev.stream()
            _lib.check(lib.tk_graph_capture_begin(s), "tk_graph_capture_begin")
            try:
                self._record_level(self.start, body_stream)
            except Exception:
                g = ctypes.c_void_p()
                lib.tk_graph_capture_end(s, ctypes.byref(g))
                raise
            finally:
                dev.INSTR.counting = counting
            _lib.check(lib.tk_graph_capture_end(s, ctypes.byref(ex)), "tk_graph_capture_end")
        self.exec = ex.value
        self._streams = (cap_stream, body_stream)
        self.launches = self._count_launches()

    def _count_launches(self) -> int:
        """Kernels of one replay outside the coarse loop + per coarse iteration
        (for the bench's gpu_launches claim)."""
        h = self.h
        a = h.levels[-1].kkt
        sgs = dev._launches("tk_forward_subst", (a.lref,)) + (
            dev._launches("tk_sgs_back_half", (a.lref,)) if self._fused_back_half(a) else
            1 + dev._launches("tk_backward_subst", (a.lref,)))
        zb = 1 if self.Z is not None else 0
        self.per_coarse_iter = sgs + zb + 1 + 1 + 1     # prec, (store z), apply, arnoldi, givens
        from .multigrid import fused_jacobi0_ok
        fixed = 0
        from .multigrid import fused_v11_ok, fused_vnn_ok
        for l in range(self.start, h.n_levels - 1):     # sweeps, restrict, prolong
            fused = h.sweeps == 1 and fused_jacobi0_ok(h.levels[l].kkt, h.omega)
            if fused and fused_v11_ok(h, h.levels[l].kkt):
                fixed += 2
                continue
            if h.sweeps > 1 and fused_vnn_ok(h, h.levels[l].kkt):
                fixed += 2 * h.sweeps
                continue
            fixed += 2 * h.sweeps + (0 if fused else 1) + 1
        fixed += 2 + 1 + 1 + 2 + (0 if zb else sgs) + 1 + 1 + 2 * 2 + 1  # begin, combine, (prec), apply, finish
        return fixed

    # --- replay -------------------------------------------------------------
    def run(self, stream=None) -> None:
        """Launch the recorded levels (input B[start], output E[start]) on the
        current stream (asynchronous; see result())."""
        s = dev.stream() if stream is None else stream
        dev.call("tk_graph_launch", self.exec, s)

    def result(self) -> int:
        """Synchronise; the coarse iteration count, or -1 when the host path
        has to redo the solve."""
        torch.cuda.current_stream().synchronize()
        if int(self.res.host[0]) != 0:
            return -1
        return int(self.res.host[1])

    def __del__(self):
        try:
            if self.exec:
                _lib.load().tk_graph_destroy(ctypes.c_void_p(self.exec))
        except Exception:
            pass


def graphed_vcycle(h, b):
    """One V-cycle from zero on device tensor b through the graph; returns
    the fine-level result, or None when the eager path must run instead."""
    from .multigrid import JACOBI0_RESIDUAL, fused_jacobi0_ok
    from .smoothers import jacobi_sweeps
    g = getattr(h, "_graph", None)
    key = (h.sweeps, float(h.omega), float(h.coarse_tol), int(h.coarse_max_iters))
    if g is None or g.key != key:
        if not getattr(h, "_graph_warm", False):
            return None                  # first cycle eager: kernel attributes, factors
        h._graph = None
        g = h._graph = VCycleGraph(h)
    a = h.levels[0].kkt
    from .multigrid import fused_v11_ok, fused_vnn_ok
    v11 = fused_v11_ok(h, a) and fused_jacobi0_ok(a, h.omega)
    vnn = (not v11) and h.sweeps > 1 and fused_vnn_ok(h, a)
    if v11:
        x = dev.empty(a.dim)
        dev.call("tk_jacobi0_restrict_um", a.lref, dev.P(b), dev.P(x), dev.P(g.B[1]),
                 dev.stream())
    elif vnn:
        xi = jacobi_sweeps(a, b, None, h.sweeps - 1, 1.0)
        x = dev.empty(a.dim)
        dev.call("tk_jacobi_restrict", a.lref, dev.P(b), dev.P(xi), dev.P(x), dev.P(g.B[1]),
                 dev.stream())
        del xi
    elif h.sweeps == 1 and JACOBI0_RESIDUAL and fused_jacobi0_ok(a, h.omega):
        x = dev.empty(a.dim)
        dev.call("tk_jacobi0_restrict", a.lref, dev.P(b), float(h.omega), dev.P(x),
                 dev.P(g.B[1]), dev.stream())
    elif h.sweeps == 1 and JACOBI0_RESIDUAL:
        x = jacobi_sweeps(a, b, None, h.sweeps, h.omega)
        dev.call("tk_residual_restrict_jacobi0", a.lref, dev.P(b), dev.P(x), float(h.omega),
                 dev.P(g.B[1]), dev.stream())
    else:
        x = jacobi_sweeps(a, b, None, h.sweeps, h.omega)
        work = dev.empty(a.dim)
        dev.call("tk_residual_restrict", a.lref, dev.P(b), dev.P(x), dev.P(g.B[1]),
                 dev.P(work), dev.stream())
        del work
    g.run()
    if dev.INSTR.counting:
        dev.INSTR.launches += g.launches
    if v11 or vnn:
        y = dev.empty(a.dim)
        dev.call("tk_jacobi_prolong", a.lref, dev.P(b), dev.P(x), dev.P(g.E[1]), dev.P(y),
                 dev.stream())
        x = jacobi_sweeps(a, b, y, h.sweeps - 1, 1.0) if vnn else y
    else:
        h.transfers[0].prolong_add(g.E[1], x)
        x = jacobi_sweeps(a, b, x, h.sweeps, h.omega)
    its = g.result()
    if its < 0:
        return None
    if dev.INSTR.counting:
        dev.INSTR.launches += its * g.per_coarse_iter
    h.stats.calls += 1
    h.stats.iters += its
    return x


def graphed_coarse(h, r):
    """SGS-GMRES coarse solve from zero (multigrid.py:245-260) as one graph
    launch; None when the host-driven solver must run instead."""
    L = h.n_levels
    g = getattr(h, "_cgraph", None)
    key = (h.sweeps, float(h.omega), float(h.coarse_tol), int(h.coarse_max_iters))
    if g is None or g.key != key:
        if not getattr(h, "_coarse_warm", False):
            return None                  # first solve eager: kernel attributes
        h._cgraph = None
        g = h._cgraph = VCycleGraph(h, start=L - 1)
    g.B[L - 1].copy_(r)
    g.run()
    if dev.INSTR.counting:
        dev.INSTR.launches += g.launches
    its = g.result()
    if its < 0:
        return None
    if dev.INSTR.counting:
        dev.INSTR.launches += its * g.per_coarse_iter
    h.stats.calls += 1
    h.stats.iters += its
    return g.E[L - 1].clone()
