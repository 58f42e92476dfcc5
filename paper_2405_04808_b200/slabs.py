"""Time-slab sharding of the multigrid-in-time hierarchy over ranks.

Row (e) of DESIGN.md.  One process per GPU; rank k owns the contiguous block
rows [b_k, b_{k+1}) of every sharded level (b_k = k*N_l/R, the last rank also
owns row N_l), so restriction is rank-local.  Per operator apply / Jacobi
sweep a rank exchanges one u segment and one mu segment with each neighbour
(the continuity couplings, kkt.py:221-247); prolongation exchanges the
neighbours' edge coarse (u, lam) / (v, mu) segments; the coarsest level is
gathered onto rank 0, solved there by the serial-in-time SGS-GMRES
(multigrid.py:245-260) and the correction scattered back; Krylov dots are
local partial sums + one allreduce.

Communication goes through a small ``Comm`` interface: ``TorchComm`` wraps
torch.distributed (NCCL on GPUs, gloo on CPU for the tests) and
``ThreadComm`` runs R virtual ranks as threads of one process (used to test
the slab kernels on a single GPU).  The local compute is a ``Backend``;
``CudaBackend`` drives libtempokkt_b200.so.
"""

from __future__ import annotations

import math
import threading
import time
from dataclasses import dataclass
from typing import List, Optional

import numpy as np
import torch

from .errors import ConfigError


# --------------------------------------------------------------------------- plan
@dataclass
class SlabPlan:
    """Row partition of every level; the coarsest level is gathered."""

    n_steps: int
    levels: int
    world: int

    def __post_init__(self):
        for lvl in range(self.levels - 1):
            nl = self.n_steps >> lvl
            if nl % self.world or (nl // self.world) % 2:
                raise ConfigError(
                    f"level {lvl}: {nl} steps cannot be split into {self.world} even slabs")

    def n_at(self, lvl: int) -> int:
        return self.n_steps >> lvl

    def rows(self, lvl: int, rank: int):
        nl = self.n_at(lvl)
        per = nl // self.world
        r0 = rank * per
        r1 = nl + 1 if rank == self.world - 1 else (rank + 1) * per
        return r0, r1

    @property
    def gather_level(self) -> int:
        return self.levels - 1


def row_start(n, nu, nz, i):
    return 0 if i == 0 else (2 * nu + nz) + (i - 1) * (4 * nu + nz)


def slab_span(n, nu, nz, r0, r1):
    a = row_start(n, nu, nz, r0)
    b = n * (4 * nu + nz) if r1 >= n + 1 else row_start(n, nu, nz, r1)
    return a, b - a


def seg_offset(n, nu, nz, r0, kind, row):
    """Local offset (within the slab starting at row r0) of segment `kind` of `row`."""
    start = row_start(n, nu, nz, row) - row_start(n, nu, nz, r0)
    if row == 0:
        off = {"u": 0, "z": nu, "lam": nu + nz}[kind]
    elif row == n:
        off = {"v": 0, "mu": nu}[kind]
    else:
        off = {"v": 0, "u": nu, "z": 2 * nu, "mu": 2 * nu + nz, "lam": 3 * nu + nz}[kind]
    return start + off


# --------------------------------------------------------------------------- comm
class Comm:
    rank: int
    size: int

    def exchange(self, send_prev, send_next, recv_prev, recv_next):  # pragma: no cover
        raise NotImplementedError

    def allreduce_sum(self, t: torch.Tensor) -> torch.Tensor:  # pragma: no cover
        raise NotImplementedError

    def allreduce_max(self, v: float) -> float:  # pragma: no cover
        raise NotImplementedError

    def gather(self, t: torch.Tensor, sizes: List[int]):  # pragma: no cover
        raise NotImplementedError

    def scatter(self, full: Optional[torch.Tensor], sizes: List[int], like: torch.Tensor):
        raise NotImplementedError  # pragma: no cover


class TorchComm(Comm):
    """torch.distributed: neighbour P2P, allreduce, gather/scatter via P2P."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)

    def exchange(self, send_prev, send_next, recv_prev, recv_next):
        d = self.dist
        ops = []
        if self.rank > 0:
            ops.append(d.P2POp(d.isend, send_prev.contiguous(), self.rank - 1, self.group))
            ops.append(d.P2POp(d.irecv, recv_prev, self.rank - 1, self.group))
        if self.rank < self.size - 1:
            ops.append(d.P2POp(d.isend, send_next.contiguous(), self.rank + 1, self.group))
            ops.append(d.P2POp(d.irecv, recv_next, self.rank + 1, self.group))
        if ops:
            for r in d.batch_isend_irecv(ops):
                r.wait()

    def allreduce_sum(self, t):
        self.dist.all_reduce(t, group=self.group)
        return t

    def allreduce_max(self, v):
        t = torch.tensor([v], dtype=torch.float64,
                         device="cuda" if torch.cuda.is_available() and
                         self.dist.get_backend(self.group) == "nccl" else "cpu")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return float(t.item())

    def gather(self, t, sizes):
        """Every rank's slab of the coarse vector onto rank 0: ONE grouped
        P2P batch (ncclGroupStart/End: the receives land side by side in the
        full vector, all in flight at once), no staging copies."""
        d = self.dist
        if self.size == 1:
            return t
        if self.rank == 0:
            offs = np.concatenate([[0], np.cumsum(sizes)])
            full = torch.empty(int(offs[-1]), dtype=t.dtype, device=t.device)
            full[:sizes[0]].copy_(t)
            ops = [d.P2POp(d.irecv, full[offs[r]:offs[r + 1]], r, self.group)
                   for r in range(1, self.size)]
            for q in d.batch_isend_irecv(ops):
                q.wait()
            return full
        for q in d.batch_isend_irecv([d.P2POp(d.isend, t.contiguous(), 0, self.group)]):
            q.wait()
        return None

    def scatter(self, full, sizes, like):
        d = self.dist
        if self.size == 1:
            return full
        if self.rank == 0:
            offs = np.concatenate([[0], np.cumsum(sizes)])
            ops = [d.P2POp(d.isend, full[offs[r]:offs[r + 1]], r, self.group)
                   for r in range(1, self.size)]
            for q in d.batch_isend_irecv(ops):
                q.wait()
            return full[:sizes[0]]
        buf = torch.empty(sizes[self.rank], dtype=like.dtype, device=like.device)
        for q in d.batch_isend_irecv([d.P2POp(d.irecv, buf, 0, self.group)]):
            q.wait()
        return buf


class _Mailbox:
    def __init__(self, size):
        self.size = size
        self.barrier = threading.Barrier(size)
        self.slots = {}
        self.lock = threading.Lock()


class ThreadComm(Comm):
    """R virtual ranks as threads of one process (single-GPU slab tests)."""

    def __init__(self, box: _Mailbox, rank: int):
        self.box = box
        self.rank = rank
        self.size = box.size

    @staticmethod
    def group(size):
        box = _Mailbox(size)
        return [ThreadComm(box, r) for r in range(size)]

    def _put(self, key, val):
        with self.box.lock:
            self.box.slots[key] = val

    def _get(self, key):
        with self.box.lock:
            return self.box.slots.pop(key)

    def exchange(self, send_prev, send_next, recv_prev, recv_next):
        if self.rank > 0:
            self._put(("x", self.rank, self.rank - 1), send_prev.clone())
        if self.rank < self.size - 1:
            self._put(("x", self.rank, self.rank + 1), send_next.clone())
        self.box.barrier.wait()
        if self.rank > 0:
            recv_prev.copy_(self._get(("x", self.rank - 1, self.rank)))
        if self.rank < self.size - 1:
            recv_next.copy_(self._get(("x", self.rank + 1, self.rank)))
        self.box.barrier.wait()

    def allreduce_sum(self, t):
        self._put(("s", self.rank), t.clone())
        self.box.barrier.wait()
        tot = sum(self.box.slots[("s", r)] for r in range(self.size))
        self.box.barrier.wait()
        if self.rank == 0:
            for r in range(self.size):
                self.box.slots.pop(("s", r))
        t.copy_(tot)
        self.box.barrier.wait()
        return t

    def allreduce_max(self, v):
        self._put(("m", self.rank), v)
        self.box.barrier.wait()
        m = max(self.box.slots[("m", r)] for r in range(self.size))
        self.box.barrier.wait()
        if self.rank == 0:
            for r in range(self.size):
                self.box.slots.pop(("m", r))
        self.box.barrier.wait()
        return m

    def gather(self, t, sizes):
        self._put(("g", self.rank), t.clone())
        self.box.barrier.wait()
        out = None
        if self.rank == 0:
            out = torch.cat([self._get(("g", r)) for r in range(self.size)])
        self.box.barrier.wait()
        return out

    def scatter(self, full, sizes, like):
        if self.rank == 0:
            offs = np.concatenate([[0], np.cumsum(sizes)])
            for r in range(self.size):
                self._put(("c", r), full[offs[r]:offs[r + 1]].clone())
        self.box.barrier.wait()
        out = self._get(("c", self.rank))
        self.box.barrier.wait()
        return out


def run_threads(comms, fn):
    """Run fn(comm) on every virtual rank; returns the per-rank results."""
    res = [None] * len(comms)
    err = []

    def body(c):
        try:
            res[c.rank] = fn(c)
        except BaseException as exc:  # pragma: no cover - surfaced below
            err.append(exc)
            c.box.barrier.abort()

    ths = [threading.Thread(target=body, args=(c,)) for c in comms]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    if err:
        raise err[0]
    return res


# --------------------------------------------------------------------------- backend
class CudaBackend:
    """Local slab compute through libtempokkt_b200.so."""

    def __init__(self):
        from . import device as dev
        from .krylov import VecOps
        self.dev = dev
        self.ops = VecOps()     # private reduction buffers (virtual ranks share a process)

    # level construction -------------------------------------------------
    def slab_level(self, p, dt, u, v, z, rows):
        from .kkt import BlockTriKKT, build_stage_blocks
        a = BlockTriKKT(build_stage_blocks(p, dt, u, v, z, rows=rows))
        a.ensure_records()
        return a

    def full_coarse(self, p, dt, u, v, z, coarse_tol, coarse_max_iters):
        from .kkt import DiagonalSolver, assemble_kkt, build_stage_blocks
        from .multigrid import MgHierarchy, MgLevel
        st = build_stage_blocks(p, dt, u, v, z)
        a = assemble_kkt(st)
        a.ensure_records()
        a.ensure_subst()
        return MgHierarchy(levels=[MgLevel(st.n_steps, dt, st, a, DiagonalSolver(a))],
                           transfers=[], coarse_tol=coarse_tol,
                           coarse_max_iters=coarse_max_iters)

    # vectors ---------------------------------------------------------------
    def to_local(self, x):
        return self.dev.to_device(x)

    def empty(self, n):
        return self.dev.empty(n)

    def zeros(self, n):
        return self.dev.zeros(n)

    # operations on a slab level `a` -----------------------------------------
    def halos(self, a):
        return a.halo_u, a.halo_mu

    def jacobi(self, a, b, x, omega):
        out = self.dev.empty(a.dim)
        self.dev.call("tk_jacobi_sweep", a.lref, self.dev.P(b), self.dev.P(x), self.dev.P(out),
                      omega, self.dev.stream())
        return out

    def apply(self, a, x):
        y = self.dev.empty(a.dim)
        self.dev.call("tk_kkt_apply", a.lref, self.dev.P(x), self.dev.P(y), self.dev.stream())
        return y

    def residual_restrict(self, a, b, x, coarse_len, jacobi0_omega=None):
        rc = self.dev.empty(coarse_len)
        if jacobi0_omega is not None:   # x = one sweep from zero: coupling terms only
            self.dev.call("tk_residual_restrict_jacobi0", a.lref, self.dev.P(b), self.dev.P(x),
                          float(jacobi0_omega), self.dev.P(rc), self.dev.stream())
            return rc
        work = self.dev.empty(a.dim)
        self.dev.call("tk_residual_restrict", a.lref, self.dev.P(b), self.dev.P(x),
                      self.dev.P(rc), self.dev.P(work), self.dev.stream())
        return rc

    def prolong_add(self, a, ec, hprev, hnext, x):
        self.dev.call("tk_prolong_add_slab", a.n_steps, a.n_u, a.n_z, a.row0,
                      a.row1 if a.row1 <= a.n_steps else a.n_steps + 1, self.dev.P(ec),
                      self.dev.P(hprev), self.dev.P(hnext), self.dev.P(x), self.dev.stream())

    # the fused V(1,1) pair on a slab (omega = 1, one sweep) ------------------
    def fused_pair_ok(self, a) -> bool:
        from . import _lib, multigrid
        if not (multigrid.FUSED_PROLONG and multigrid.FUSED_JACOBI0 and multigrid.JACOBI0_RESIDUAL):
            return False
        return bool(_lib.load().tk_jacobi_prolong_ok(a.lref, 1.0))

    def jacobi0_restrict_um(self, a, b, coarse_len):
        """Zero-start sweep (u / mu segments of x only) + the coarse entries its
        own rows feed; restrict_fix completes rc after the halo exchange of x."""
        x, rc = self.dev.empty(a.dim), self.dev.empty(coarse_len)
        self.dev.call("tk_jacobi0_restrict_um", a.lref, self.dev.P(b), self.dev.P(x),
                      self.dev.P(rc), self.dev.stream())
        return x, rc

    def restrict_fix(self, a, rc):
        self.dev.call("tk_restrict_fix_slab", a.lref, self.dev.P(rc), self.dev.stream())

    def jacobi_restrict(self, a, b, x_in, coarse_len):
        """An omega = 1 sweep from x_in (its halos exchanged) + the coarse entries
        its own rows feed; restrict_fix_x(…, 1) before and (…, 2) after the halo
        exchange of the result complete rc."""
        x, rc = self.dev.empty(a.dim), self.dev.empty(coarse_len)
        self.dev.call("tk_jacobi_restrict", a.lref, self.dev.P(b), self.dev.P(x_in),
                      self.dev.P(x), self.dev.P(rc), self.dev.stream())
        return x, rc

    def restrict_fix_x(self, a, rc, phase):
        self.dev.call("tk_restrict_fix_slab_x", a.lref, self.dev.P(rc), int(phase),
                      self.dev.stream())

    def jacobi_prolong(self, a, b, x, ec, chalo):
        y = self.dev.empty(a.dim)
        self.dev.call("tk_jacobi_prolong_slab", a.lref, self.dev.P(b), self.dev.P(x),
                      self.dev.P(ec), self.dev.P(chalo), self.dev.P(y), self.dev.stream())
        return y

    def coarse_solve(self, h, r):
        from .multigrid import coarse_solve
        return coarse_solve(h, r)

    def local_dot(self, x, y):
        return self.ops.dot_dev(x, y).reshape(1).clone()

    # Krylov vector operations on slab vectors (SlabSpace) ---------------------
    def scale_into(self, a, x, y):
        self.ops.scale_into(a, x, y)

    def axpy(self, a, x, y):
        self.ops.axpy(a, x, y)

    def rsub(self, b, y):
        self.dev.call("tk_rsub", y.numel(), self.dev.P(b), self.dev.P(y), self.dev.stream())

    def gemv_t_add(self, V, c, x):
        self.ops.gemv_t_add(V, c, x)

    def sq_norms(self, vecs):
        """Local squared norms of `vecs` side by side in one device tensor."""
        out = self.dev.empty(len(vecs))
        for k, v in enumerate(vecs):
            self.dev.call("tk_dot", v.numel(), self.dev.P(v), self.dev.P(v),
                          out[k:].data_ptr(), self.dev.P(self.ops.work), self.dev.stream())
        return out

    def mgs(self, comm, V, j, w):
        """One modified Gram-Schmidt Arnoldi step on slab vectors (krylov.py:
        141-163): every h_i = <V_i, w> is a local partial dot + an allreduce
        that stays on the device and feeds `w -= h_i V_i` (tk_axpy_dev), the
        norm likewise (tk_sqrt_div writes V_{j+1} = w / h_{j+1}); the host
        reads the column once, after the whole step has been enqueued."""
        d = self.dev
        n = w.numel()
        if getattr(self, "_h", None) is None or self._h.numel() < j + 3:
            self._h = d.empty(max(64, 2 * (j + 3)))   # h_0..h_{j+1} + the squared-norm slot
        h = self._h
        for i in range(j + 1):
            d.call("tk_dot", n, d.P(V[i]), d.P(w), h[i:].data_ptr(), d.P(self.ops.work),
                   d.stream())
            comm.allreduce_sum(h[i:i + 1])
            d.call("tk_axpy_dev", n, h[i:].data_ptr(), -1.0, d.P(V[i]), d.P(w), d.stream())
        # the squared norm in a scratch slot: tk_sqrt_div reads sq[0] in every CTA
        # while one thread stores the root, so the two must not alias
        sq = h[h.numel() - 1:]
        d.call("tk_dot", n, d.P(w), d.P(w), sq.data_ptr(), d.P(self.ops.work), d.stream())
        comm.allreduce_sum(sq)
        d.call("tk_sqrt_div", n, sq.data_ptr(), h[j + 1:].data_ptr(), d.P(w),
               d.P(V[j + 1]), d.stream())
        return h[:j + 2].cpu().numpy()

    def finish(self):
        pass


# --------------------------------------------------------------------------- hierarchy
class SlabHierarchy:
    """Per-rank part of the time-sharded V-cycle hierarchy."""

    def __init__(self, p, u, v, z, grid, levels, comm: Comm, sweeps=1, omega=1.0,
                 coarse_tol=1e-2, coarse_max_iters=401, backend=None):
        if levels < 2:
            raise ConfigError("the sharded hierarchy needs >= 2 levels")
        self.p, self.comm = p, comm
        self.be = backend or CudaBackend()
        self.plan = SlabPlan(grid.n_steps, levels, comm.size)
        self.sweeps, self.omega = sweeps, omega
        self.nu, self.nz = p.n_u, p.n_z
        self.levels = []
        u, v, z = (np.asarray(a, dtype=np.float64) for a in (u, v, z))
        dt = grid.dt
        for lvl in range(levels - 1):
            rows = self.plan.rows(lvl, comm.rank)
            self.levels.append(self.be.slab_level(p, dt, u, v, z, rows))
            u, v, z = u[1::2], v[1::2], 0.5 * (z[0::2] + z[1::2])
            dt *= 2.0
        self.nc = self.plan.n_at(levels - 1)
        self.coarse = None
        if comm.rank == 0:
            self.coarse = self.be.full_coarse(p, dt, u, v, z, coarse_tol, coarse_max_iters)
        # coarse slab sizes for gather/scatter
        self.coarse_sizes = [slab_span(self.nc, self.nu, self.nz,
                                       *self._coarse_rows(levels - 2, r))[1]
                             for r in range(comm.size)]

    # geometry -------------------------------------------------------------
    def _coarse_rows(self, lvl, rank):
        r0, r1 = self.plan.rows(lvl, rank)
        nl = self.plan.n_at(lvl)
        return r0 // 2, (nl // 2 + 1) if r1 == nl + 1 else r1 // 2

    @property
    def local_dim(self):
        return self.levels[0].dim

    def local_span(self):
        a = self.levels[0]
        return slab_span(a.n_steps, self.nu, self.nz, a.row0, a.row1)

    # halo exchanges -----------------------------------------------------------
    def exchange_x(self, lvl, x):
        a = self.levels[lvl]
        n, nu, nz, c = a.n_steps, self.nu, self.nz, self.comm
        hu, hm = self.be.halos(a)
        send_prev = send_next = None
        if c.rank > 0:
            o = seg_offset(n, nu, nz, a.row0, "mu", a.row0)
            send_prev = x[o:o + nu]
        if c.rank < c.size - 1:
            o = seg_offset(n, nu, nz, a.row0, "u", a.row1 - 1)
            send_next = x[o:o + nu]
        c.exchange(send_prev, send_next, hu, hm)

    def exchange_coarse(self, lvl, ec):
        """Return (hprev = prev slab's last coarse (u, lam), hnext = next's first (v, mu))."""
        c, nu, nz = self.comm, self.nu, self.nz
        nc = self.plan.n_at(lvl + 1)
        c0, c1 = self._coarse_rows(lvl, c.rank)
        both = self.be.zeros(4 * nu)      # one buffer: tk_jacobi_prolong_slab's chalo
        hprev, hnext = both[:2 * nu], both[2 * nu:]
        self._chalo = both
        send_prev = send_next = None
        if c.rank > 0:
            ov = seg_offset(nc, nu, nz, c0, "v", c0)
            om = seg_offset(nc, nu, nz, c0, "mu", c0)
            send_prev = torch.cat([ec[ov:ov + nu], ec[om:om + nu]])
        if c.rank < c.size - 1:
            ou = seg_offset(nc, nu, nz, c0, "u", c1 - 1)
            ol = seg_offset(nc, nu, nz, c0, "lam", c1 - 1)
            send_next = torch.cat([ec[ou:ou + nu], ec[ol:ol + nu]])
        c.exchange(send_prev, send_next, hprev, hnext)
        return hprev, hnext

    # the V-cycle ------------------------------------------------------------
    def _smooth(self, lvl, b, x, sweeps):
        a = self.levels[lvl]
        for _ in range(sweeps):
            if x is not None:
                self.exchange_x(lvl, x)
            x = self.be.jacobi(a, b, x, self.omega)
        return x

    def _cycle(self, lvl, b):
        a = self.levels[lvl]
        c0, c1 = self._coarse_rows(lvl, self.comm.rank)
        nc = self.plan.n_at(lvl + 1)
        clen = slab_span(nc, self.nu, self.nz, c0, c1)[1]
        from . import multigrid
        fp = getattr(self.be, "fused_pair_ok", None)
        if self.sweeps == 1 and float(self.omega) == 1.0 and fp is not None and fp(a):
            # V(1,1), omega = 1: pre-smoothing + restriction and prolongation +
            # post-smoothing as the two fused kernels (multigrid._cycle's v11 path);
            # the one exchange of x serves the coarse boundary entries and the
            # post-smoothing couplings
            x, rc = self.be.jacobi0_restrict_um(a, b, clen)
            self.exchange_x(lvl, x)
            self.be.restrict_fix(a, rc)
            ec = self._coarse_correction(lvl, rc)
            self.exchange_coarse(lvl, ec)
            return self.be.jacobi_prolong(a, b, x, ec, self._chalo)
        if self.sweeps > 1 and float(self.omega) == 1.0 and fp is not None and fp(a):
            # several sweeps (multigrid._cycle's vnn path): the LAST pre-smoothing
            # sweep writes the restricted residual (x_in - x at the couplings; the two
            # boundary segments from the halos of x_in, then of x), the FIRST
            # post-smoothing sweep takes the prolongation
            x_in = self._smooth(lvl, b, None, self.sweeps - 1)
            self.exchange_x(lvl, x_in)
            x, rc = self.be.jacobi_restrict(a, b, x_in, clen)
            self.be.restrict_fix_x(a, rc, 1)
            self.exchange_x(lvl, x)
            self.be.restrict_fix_x(a, rc, 2)
            del x_in
            ec = self._coarse_correction(lvl, rc)
            self.exchange_coarse(lvl, ec)
            y = self.be.jacobi_prolong(a, b, x, ec, self._chalo)
            return self._smooth(lvl, b, y, self.sweeps - 1)
        x = self._smooth(lvl, b, None, self.sweeps)
        self.exchange_x(lvl, x)
        j0 = self.omega if (self.sweeps == 1 and multigrid.JACOBI0_RESIDUAL and
                            getattr(self.be, "jacobi0", True)) else None
        rc = self.be.residual_restrict(a, b, x, clen, j0)
        ec = self._coarse_correction(lvl, rc)
        hprev, hnext = self.exchange_coarse(lvl, ec)
        self.be.prolong_add(a, ec, hprev, hnext, x)
        return self._smooth(lvl, b, x, self.sweeps)

    def _coarse_correction(self, lvl, rc):
        if lvl + 1 == len(self.levels):
            full = self.comm.gather(rc, self.coarse_sizes)
            ef = self.be.coarse_solve(self.coarse, full) if self.comm.rank == 0 else None
            return self.comm.scatter(ef, self.coarse_sizes, rc)
        return self._cycle(lvl + 1, rc)

    def vcycle(self, b_local):
        return self._cycle(0, b_local)

    # distributed operator and dots (for (F)GMRES on the slabs) ---------------
    def apply(self, x):
        self.exchange_x(0, x)
        return self.be.apply(self.levels[0], x)

    def dot(self, x, y) -> float:
        t = self.be.local_dot(x, y)
        return float(self.comm.allreduce_sum(t).item())


# --------------------------------------------------------------------------- Krylov
class SlabSpace:
    """Vector space of a time-sharded (F)GMRES (the ``space`` of
    krylov._gmres_engine): vectors are per-rank slabs, axpy-type operations are
    local, every inner product is a local partial sum + one allreduce, so all
    ranks see the same Hessenberg column and take the same branches
    (reference krylov.py:77-191 run on vectors that happen to be sharded)."""

    def __init__(self, hier: "SlabHierarchy"):
        self.h, self.be, self.comm = hier, hier.be, hier.comm

    def to_local(self, x):
        return self.be.to_local(x)

    def _norms(self, vecs):
        sq = self.comm.allreduce_sum(self.be.sq_norms(vecs))
        return [math.sqrt(v) for v in sq.tolist()]

    def nrm2(self, x) -> float:
        return self._norms([x])[0]

    def nrm2_pair(self, x, r):
        a, b = self._norms([x, r])
        return a, b

    def scale_into(self, a, x, y):
        self.be.scale_into(a, x, y)

    def axpy(self, a, x, y):
        self.be.axpy(a, x, y)

    def arnoldi(self, V, j, w):
        return self.be.mgs(self.comm, V, j, w)

    def gemv_t_add(self, V, c, x):
        self.be.gemv_t_add(V, c, x)

    def residual(self, op, b, x):
        y = self.be.to_local(op(x))
        self.be.rsub(b, y)
        return y

    def finish(self):
        self.be.finish()


def slab_operator(h: SlabHierarchy):
    """The time-sharded augmented operator as a krylov.LinearOperator on slab
    vectors (BlockTriKKT.as_operator, kkt.py:249-250, with the halo exchange)."""
    from .krylov import LinearOperator
    return LinearOperator(dim=h.local_dim, apply=h.apply)


def slab_preconditioner(h: SlabHierarchy):
    """One sharded V-cycle from zero (mg_preconditioner, multigrid.py:304-311)."""
    from .krylov import Preconditioner
    return Preconditioner(apply=h.vcycle, is_flexible=True)


def fgmres(h: SlabHierarchy, b_local, x0=None, rel_tol=1e-10, max_iters=401, restart=None):
    """Flexible GMRES (krylov.py:204-210) over time slabs: this rank's part of
    the solution and the (rank-identical) SolveReport."""
    from .krylov import _gmres_engine
    return _gmres_engine(slab_operator(h), slab_preconditioner(h), b_local, x0, rel_tol,
                         max_iters, restart, flexible=True, space=SlabSpace(h))


def gmres(h: SlabHierarchy, prec, b_local, x0=None, rel_tol=1e-10, max_iters=401, restart=None):
    """Restarted right-preconditioned GMRES (krylov.py:194-201) over time
    slabs with a fixed (linear) slab preconditioner, or None."""
    from .krylov import _gmres_engine
    return _gmres_engine(slab_operator(h), prec, b_local, x0, rel_tol, max_iters, restart,
                         flexible=False, space=SlabSpace(h))


# --------------------------------------------------------------------------- bench
def bench_rank(args, rank, world, local_rank):
    """bench.py --gpus N (N > 1): strong scaling of the V-cycle on configs[idx]."""
    import torch.distributed as dist

    from . import configs
    from . import device as dev
    if not dist.is_initialized():
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    comm = TorchComm()
    s = configs.build_setup(args.config)
    S = s.solver
    h = SlabHierarchy(s.problem, s.u, s.v, s.z, s.grid, s.levels, comm, sweeps=S["sweeps"],
                      omega=S["omega"], coarse_tol=S["coarse_tol"],
                      coarse_max_iters=S["coarse_max_iters"])
    off, ln = h.local_span()
    rhs = s.rhs()
    r_host = torch.from_numpy(np.ascontiguousarray(rhs[off:off + ln])).pin_memory()
    r_loc = dev.to_device(r_host)
    for _ in range(max(args.warmup, 1)):
        h.vcycle(r_loc)
    torch.cuda.synchronize()
    dist.barrier()
    clk = None
    if rank == 0:
        from bench import ClockSampler
        clk = ClockSampler(local_rank)
        clk.start()
        time.sleep(0.3)
    dev.INSTR.counting, dev.INSTR.launches = True, 0
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    dist.barrier()
    e0.record()
    for _ in range(args.steps):
        h.vcycle(r_loc)
    e1.record()
    torch.cuda.synchronize()
    dist.barrier()
    dev.INSTR.counting = False
    ms = comm.allreduce_max(e0.elapsed_time(e1)) / args.steps
    launches = int(comm.allreduce_max(float(dev.INSTR.launches)))
    clocks = clk.stop() if clk else None
    # roofline of the dominant kernel: this rank's fine-level Jacobi sweep over
    # its slab (x present), CUDA events on the launching stream, slowest rank
    from . import roofline
    a0 = h.levels[0]
    x0 = h.be.jacobi(a0, r_loc, None, 1.0)
    h.exchange_x(0, x0)
    for _ in range(2):
        h.be.jacobi(a0, r_loc, x0, 1.0)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        h.be.jacobi(a0, r_loc, x0, 1.0)
    e1.record()
    torch.cuda.synchronize()
    jms = comm.allreduce_max(e0.elapsed_time(e1) / 5)
    # algorithmic bytes of the slab (omega = 1: the splitting-form sweep reads b, the
    # two coupling segments of x per row and this slab's stage data, writes x out)
    rows = min(a0.row1, a0.n_steps) - a0.row0
    sb = roofline.stage_bytes(a0) * rows // a0.n_steps
    jbytes = 8 * a0.dim * 2 + 16 * rows * a0.n_u + sb
    try:
        import json as _json
        import os as _os
        with open(_os.path.join(_os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))),
                               "MEASURED_PEAKS.json")) as fh:
            peak, peak_kind = float(_json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        peak, peak_kind = 6650.0, "fallback"
    ach = jbytes / (jms * 1e-3) / 1e9
    # e2e: pinned host slice -> device, V-cycle, device -> pinned host, per rank
    out_host = torch.empty(ln, dtype=torch.float64).pin_memory()
    e2e_steps = max(2, min(args.steps, 5))
    torch.cuda.synchronize()
    dist.barrier()
    e0.record()
    for _ in range(e2e_steps):
        r_loc.copy_(r_host, non_blocking=True)
        out_host.copy_(h.vcycle(r_loc), non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    dist.barrier()
    e2e_ms = comm.allreduce_max(e0.elapsed_time(e1)) / e2e_steps
    unknowns = s.grid.n_steps * s.dof_per_step
    # the full sharded MG-FGMRES solve (tol / iteration cap of the config), wall
    # clock between barriers with device synchronisation, slowest rank; the
    # restart length is sized to the smallest free HBM over the ranks (V and Z
    # hold two slab vectors per iteration) so that every rank restarts alike
    solve = None
    if getattr(args, "solve_config", 0) >= 0:
        torch.cuda.empty_cache()
        free, _ = torch.cuda.mem_get_info()
        m_fit = int(0.9 * free // (2 * ln * 8)) - 4
        m_fit = -int(comm.allreduce_max(-float(m_fit)))
        restart = None if m_fit >= S["max_iters"] + 1 else max(2, m_fit)
        if rank == 0:
            h.coarse.stats = type(h.coarse.stats)()
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        xs, rep = fgmres(h, r_loc, rel_tol=S["rel_tol"], max_iters=S["max_iters"],
                         restart=restart)
        torch.cuda.synchronize()
        dist.barrier()
        secs = comm.allreduce_max(time.perf_counter() - t0)
        del xs
        solve = {"config": f"configs[{args.config}] {s.describe()}", "seconds": round(secs, 4),
                 "outer": "fgmres over time slabs (distributed MGS, allreduced dots)",
                 "restart": restart, "iterations": rep.iterations,
                 "final_rel_residual": rep.final_relative_residual,
                 "coarse_iters_avg": h.coarse.stats.average if rank == 0 else None}
    if rank != 0:
        return None
    return {
        "metric": "V-cycle time-step*DoF/s (fp64) + full MG-FGMRES solve time",
        "value": unknowns / (ms * 1e-3), "unit": "time-step*DoF/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: forward-march linearisation + N(0,1) rhs (seeded)",
        "config": {"workload": f"configs[{args.config}] {s.describe()}",
                   "parallelism": f"time-slabs x{world}, coarse level gathered on rank 0",
                   "kkt_dim": s.dim, "l2": "inputs larger than L2"},
        "e2e": {"value": unknowns / (e2e_ms * 1e-3), "unit": "time-step*DoF/s",
                "h2d_bytes_per_step": int(rhs.nbytes), "d2h_bytes_per_step": int(rhs.nbytes),
                "ms_per_step": e2e_ms},
        "roofline": {"bound": "hbm", "kernel": "tk_jacobi_sweep (fine level, per-rank slab)",
                     "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                     "traffic": None, "peak_kind": peak_kind, "bytes_per_launch": jbytes,
                     "ms_per_launch": jms},
        "gpu_launches": launches,
        "clocks": clocks,
        "cpu_baseline": None,
        "solve": solve,
    }
