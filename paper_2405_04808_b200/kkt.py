"""The virtual-variable augmented (KKT) operator on the device.

Mirrors the reference module kkt.py: ``StageBlocks`` (:53-80),
``build_stage_blocks`` (:100-124), ``KktLayout`` (:127-191),
``BlockTriKKT`` (:194-276), ``assemble_kkt`` (:279-320),
``DiagonalSolver`` (:338-389).  Vectors are float64 CUDA tensors in the
reference's exact time-clustered ordering; numpy inputs are accepted and
answered with numpy (host<->device copies around the device computation).

Stage data live in HBM in one of two structure families chosen at
assembly (include/tempokkt_b200.h):

* DENSE -- n_u, n_z <= 4 (van der Pol): K, C, B as [N, nu, nu|nz];
* TRI   -- tridiagonal-in-space blocks with n_z == n_u and B = kappa*Qz
  (P1 Burgers): K, C as [N, 3, nu] diagonals.

Anything else raises :class:`UnsupportedStructure` -- there is no CPU path.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import _lib
from . import device as dev
from .errors import DimensionMismatch, UnsupportedStructure
from .timedisc import ProblemSpec, stage_jacobians, stage_weights

FAMILY_DENSE = _lib.FAMILY_DENSE
FAMILY_TRI = _lib.FAMILY_TRI
MAX_DENSE = 4


class KktLayout:
    """Index map of the time-clustered ordering (kkt.py:127-191)."""

    def __init__(self, n_steps: int, n_u: int, n_z: int):
        self.n_steps, self.n_u, self.n_z = n_steps, n_u, n_z
        self.first_size = 2 * n_u + n_z
        self.interior_size = 4 * n_u + n_z
        self.last_size = 2 * n_u
        self.dim = n_steps * (4 * n_u + n_z)
        n, nu, nz = n_steps, n_u, n_z
        starts = np.empty(n + 1, dtype=np.intp)
        starts[0] = 0
        starts[1:] = self.first_size + np.arange(n) * self.interior_size
        self.block_starts = starts
        t = np.arange(1, n + 1)
        seg = lambda off, w: off[:, None] + np.arange(w)[None, :]
        self._rows = {
            "u": seg(np.where(t == 1, 0, starts[t - 1] + nu), nu),
            "v": seg(starts[t], nu),
            "z": seg(np.where(t == 1, nu, starts[t - 1] + 2 * nu), nz),
            "lam": seg(np.where(t == 1, nu + nz, starts[t - 1] + 3 * nu + nz), nu),
            "mu": seg(np.where(t == n, starts[t] + nu, starts[t] + 2 * nu + nz), nu),
        }

    def rows(self, kind: str) -> np.ndarray:
        return self._rows[kind]

    def offset(self, kind: str, t: int) -> int:
        return int(self._rows[kind][t - 1, 0])

    def block_size(self, i: int) -> int:
        if i == 0:
            return self.first_size
        if i == self.n_steps:
            return self.last_size
        return self.interior_size

    def pack(self, u, v, z, lam, mu) -> np.ndarray:
        out = np.empty(self.dim)
        for k, a in (("u", u), ("v", v), ("z", z), ("lam", lam), ("mu", mu)):
            out[self._rows[k]] = a
        return out

    def unpack(self, x: np.ndarray):
        x = np.asarray(x)
        if x.shape != (self.dim,):
            raise DimensionMismatch(f"vector shape {x.shape} != ({self.dim},)")
        return tuple(x[self._rows[k]] for k in ("u", "v", "z", "lam", "mu"))


def _tri_diags(a: np.ndarray) -> np.ndarray:
    """[3, n] (sub, diag, sup) of a tridiagonal matrix; sub[0] = sup[-1] = 0."""
    n = a.shape[0]
    out = np.zeros((3, n))
    out[1] = np.diag(a)
    out[0, 1:] = np.diag(a, -1)
    out[2, :-1] = np.diag(a, 1)
    return out


def _is_tridiagonal(a: np.ndarray) -> bool:
    return not (np.triu(a, 2).any() or np.tril(a, -2).any())


@dataclass
class StageBlocks:
    """Per-stage linearisation data resident in HBM (kkt.py:53-80).

    ``K``, ``C`` (and ``B`` for DENSE) are per-stage device tensors;
    the weights are time-constant apart from the terminal stage
    (``Qm`` for stages < N-1, ``Ql`` for stage N-1; ``Qz`` all stages).
    """

    family: int
    n_steps: int
    n_u: int
    n_z: int
    K: torch.Tensor
    C: torch.Tensor
    B: Optional[torch.Tensor]
    Qm: torch.Tensor
    Ql: torch.Tensor
    Qz: torch.Tensor
    Qm_inv: Optional[torch.Tensor] = None
    Ql_inv: Optional[torch.Tensor] = None
    Qz_inv: Optional[torch.Tensor] = None
    kappa: float = 0.0
    qz_cr: Optional[torch.Tensor] = None
    qz_w: Optional[torch.Tensor] = None
    host_weights: dict = field(default_factory=dict, repr=False)
    # time slab: global block rows [row0, row1) of a level with n_global steps
    # (row1 == 0: the whole level); K/C/B then hold stages [row0, min(row1, N)).
    n_global: int = 0
    row0: int = 0
    row1: int = 0

    def __post_init__(self):
        if self.n_global == 0:
            self.n_global = self.n_steps

    @property
    def rows(self):
        return self.row0, (self.row1 if self.row1 > 0 else self.n_global + 1)

    @property
    def dim(self) -> int:
        r0, r1 = self.rows
        return slab_span(self.n_global, self.n_u, self.n_z, r0, r1)[1]


def row_start(n: int, nu: int, nz: int, i: int) -> int:
    """Global offset of block row i (kkt.py:144-147)."""
    return 0 if i == 0 else (2 * nu + nz) + (i - 1) * (4 * nu + nz)


def slab_span(n: int, nu: int, nz: int, r0: int, r1: int):
    """(offset, length) of block rows [r0, r1) in the global vector."""
    a = row_start(n, nu, nz, r0)
    b = n * (4 * nu + nz) if r1 >= n + 1 else row_start(n, nu, nz, r1)
    return a, b - a


def _weights(family, q_mid, q_last, q_z, kappa):
    """Upload the constant weights in the family's storage format."""
    hw = dict(q_mid=q_mid, q_last=q_last, q_z=q_z)
    if family == FAMILY_DENSE:
        return dict(Qm=dev.to_device(q_mid), Ql=dev.to_device(q_last), Qz=dev.to_device(q_z),
                    Qm_inv=dev.to_device(np.linalg.inv(q_mid)),
                    Ql_inv=dev.to_device(np.linalg.inv(q_last)),
                    Qz_inv=dev.to_device(np.linalg.inv(q_z)), kappa=0.0, qz_cr=None,
                    host_weights=hw)
    qz3 = np.ascontiguousarray(_tri_diags(q_z))
    lib = _lib.load()
    n = q_z.shape[0]
    cr = np.empty_like(qz3)
    _lib.check(lib.tk_cr_scalar_factor(n, qz3.ctypes.data, cr.ctypes.data), "tk_cr_scalar_factor")
    # (active, active) block of Qz^{-1} at the cyclic-reduction cut, transposed:
    # the inverse of the scalar system reduced onto the active nodes
    a = int(lib.tk_tri_cut_nodes(n))
    idx = np.empty(a, dtype=np.int32)
    _lib.check(lib.tk_tri_cut_indices(n, idx.ctypes.data), "tk_tri_cut_indices")
    qzw = np.ascontiguousarray(np.linalg.inv(q_z)[np.ix_(idx, idx)].T)
    return dict(Qm=dev.to_device(_tri_diags(q_mid)), Ql=dev.to_device(_tri_diags(q_last)),
                Qz=dev.to_device(qz3), kappa=float(kappa), qz_cr=dev.to_device(cr),
                qz_w=dev.to_device(qzw), host_weights=hw)


def _problem_weights(p: ProblemSpec, dt: float, n: int):
    q_mid, _, q_z = stage_weights(p, dt, 0, max(n, 2))
    q_last, _, _ = stage_weights(p, dt, n - 1, n)
    return np.ascontiguousarray(q_mid), np.ascontiguousarray(q_last), np.ascontiguousarray(q_z)


def _choose_family(n_u, n_z, q_mid, q_z, kappa_ok):
    if n_u <= MAX_DENSE and n_z <= MAX_DENSE:
        return FAMILY_DENSE
    if n_z == n_u and _is_tridiagonal(q_mid) and _is_tridiagonal(q_z) and kappa_ok:
        return FAMILY_TRI
    raise UnsupportedStructure(
        f"stage blocks with n_u={n_u}, n_z={n_z} are neither small dense (<= {MAX_DENSE}) "
        "nor tridiagonal with B = kappa*Qz")


def build_stage_blocks(p: ProblemSpec, dt: float, u_seq, v_seq, z_seq,
                       rows=None) -> StageBlocks:
    """Linearise every stage at (u, v, z) with spacing dt (kkt.py:100-124).

    Built-in problems (``p.native``) are linearised on the device by
    tk_stage_vanderpol / tk_stage_burgers; other specs go through their
    Python callables once (setup) and are uploaded.  ``rows=(r0, r1)``
    builds only the stages of the time slab of block rows [r0, r1).
    """
    n = int(np.shape(u_seq)[0])
    nu, nz = p.n_u, p.n_z
    q_mid, q_last, q_z = _problem_weights(p, dt, n)
    nat = p.native
    r0, r1 = (0, n + 1) if rows is None else (int(rows[0]), int(rows[1]))
    slab = dict(n_global=n, row0=r0, row1=0 if rows is None else r1)
    s0, s1 = r0, min(r1, n)           # stages of the slab
    ns = max(s1 - s0, 0)
    if nat is not None and nat["kind"] in ("vanderpol", "burgers"):
        u = dev.to_device(np.asarray(u_seq)[s0:s1] if not isinstance(u_seq, torch.Tensor)
                          else u_seq[s0:s1])
        v = dev.to_device(np.asarray(v_seq)[s0:s1] if not isinstance(v_seq, torch.Tensor)
                          else v_seq[s0:s1])
        first = p.u0 if s0 == 0 else (v_seq[s0 - 1])
        u0 = dev.to_device(first)
        if nat["kind"] == "vanderpol":
            z = dev.to_device(np.asarray(z_seq)[s0:s1] if not isinstance(z_seq, torch.Tensor)
                              else z_seq[s0:s1])
            K = dev.empty(max(ns, 1), nu, nu)
            Cm = dev.empty(max(ns, 1), nu, nu)
            B = dev.empty(max(ns, 1), nu, nz)
            if ns:
                dev.call("tk_stage_vanderpol", ns, dt, p.theta, nat["mu"], nz, dev.P(u0),
                         dev.P(u), dev.P(v), dev.P(z), dev.P(K), dev.P(Cm), dev.P(B),
                         dev.stream())
            w = _weights(FAMILY_DENSE, q_mid, q_last, q_z, 0.0)
            return StageBlocks(FAMILY_DENSE, ns, nu, nz, K, Cm, B, **w, **slab)
        # Burgers: F_z = M and w_control = alpha*M  =>  B = dt*M = kappa*Qz, kappa = 1/alpha
        kappa = float(p.mass[0, 0] / p.w_control[0, 0])
        K = dev.empty(max(ns, 1), 3, nu)
        Cm = dev.empty(max(ns, 1), 3, nu)
        if ns:
            dev.call("tk_stage_burgers", ns, nu, dt, p.theta, nat["nu"], dev.P(u0), dev.P(u),
                     dev.P(v), dev.P(K), dev.P(Cm), dev.stream())
        w = _weights(FAMILY_TRI, q_mid, q_last, q_z, kappa)
        return StageBlocks(FAMILY_TRI, ns, nu, nz, K, Cm, None, **w, **slab)
    # generic ProblemSpec: evaluate the callables once on the host
    u_seq, v_seq, z_seq = (np.asarray(a, dtype=np.float64) for a in (u_seq, v_seq, z_seq))
    k = np.empty((n, nu, nu)); c = np.empty((n, nu, nu)); b = np.empty((n, nu, nz))
    v_prev = np.asarray(p.u0, dtype=np.float64)
    for i in range(n):
        k[i], c[i], b[i] = stage_jacobians(p, v_prev, u_seq[i], z_seq[i], dt)
        v_prev = v_seq[i]
    qu = np.empty((n, nu, nu)); qz = np.empty((n, nz, nz))
    for i in range(n):
        qu[i], _, qz[i] = stage_weights(p, dt, i, n)
    st = stage_blocks_from_arrays(k, c, b, qu, qu, qz)
    if rows is None:
        return st
    st.K = st.K[s0:max(s1, s0 + 1)].contiguous()
    st.C = st.C[s0:max(s1, s0 + 1)].contiguous()
    if st.B is not None:
        st.B = st.B[s0:max(s1, s0 + 1)].contiguous()
    st.n_steps, st.n_global, st.row0, st.row1 = ns, n, r0, r1
    return st


def stage_blocks_from_arrays(k, c, b, q_u, q_v, q_z) -> StageBlocks:
    """Upload reference-layout StageBlocks arrays (kkt.py:63-68) after
    checking the time structure of the weights and choosing the family."""
    k, c, b, q_u, q_v, q_z = (np.ascontiguousarray(a, dtype=np.float64)
                              for a in (k, c, b, q_u, q_v, q_z))
    n, nu, nz = k.shape[0], k.shape[1], b.shape[2]
    if not np.array_equal(q_u, q_v):
        raise UnsupportedStructure("q_u and q_v must be equal (timedisc.py:206)")
    if n > 1 and not (q_u[:-1] == q_u[0]).all():
        raise UnsupportedStructure("q_u must be time-constant before the last stage")
    if not (q_z == q_z[0]).all():
        raise UnsupportedStructure("q_z must be time-constant")
    q_mid, q_last, qz = q_u[0], q_u[-1], q_z[0]
    kappa, kappa_ok = 0.0, False
    if nz == nu and qz[0, 0] != 0.0:
        kappa = float(b[0, 0, 0] / qz[0, 0])
        kappa_ok = bool(np.allclose(b, kappa * qz[None], rtol=0.0,
                                    atol=1e-13 * max(np.abs(b).max(), 1e-300)))
    fam = _choose_family(nu, nz, q_mid, qz, kappa_ok)
    if fam == FAMILY_DENSE:
        w = _weights(fam, q_mid, q_last, qz, 0.0)
        return StageBlocks(fam, n, nu, nz, dev.to_device(k), dev.to_device(c),
                           dev.to_device(b), **w)
    if not all(_is_tridiagonal(a) for a in (k[i] for i in range(n))) or \
            not all(_is_tridiagonal(a) for a in (c[i] for i in range(n))):
        raise UnsupportedStructure("K_i / C_i are not tridiagonal")
    kd = np.stack([_tri_diags(k[i]) for i in range(n)])
    cd = np.stack([_tri_diags(c[i]) for i in range(n)])
    w = _weights(fam, q_mid, q_last, qz, kappa)
    return StageBlocks(fam, n, nu, nz, dev.to_device(kd), dev.to_device(cd), None, **w)


def _toeplitz(q) -> bool:
    """TRI weight [3][n] (sub, diag, sup) with constant diagonals."""
    w = (q.detach().cpu().numpy() if isinstance(q, torch.Tensor) else np.asarray(q)).reshape(3, -1)
    if w.shape[1] < 2:
        return False
    sub, d, sup = w
    s = sup[0]
    return bool((d == d[0]).all() and (sup[:-1] == s).all() and (sub[1:] == s).all())


class BlockTriKKT:
    """Symmetric block-tridiagonal augmented operator on the device
    (kkt.py:194-276).  ``apply``/``residual``/``apply_diag`` launch the
    CUDA kernels; numpy in -> numpy out."""

    def __init__(self, stage: StageBlocks):
        self.stage = stage
        self.n_steps, self.n_u, self.n_z = stage.n_global, stage.n_u, stage.n_z
        self.row0, self.row1 = stage.rows
        self.is_slab = not (self.row0 == 0 and self.row1 == self.n_steps + 1)
        self._layout = None
        s = stage
        # halo buffers of a time slab (refreshed by the neighbour exchange)
        self.halo_u = dev.zeros(s.n_u) if self.row0 > 0 else None
        self.halo_mu = dev.zeros(s.n_u) if self.row1 <= self.n_steps else None
        self.level = _lib.TkLevel(
            family=s.family, n_steps=s.n_global, n_u=s.n_u, n_z=s.n_z,
            K=dev.P(s.K), C=dev.P(s.C), B=dev.P(s.B), Qm=dev.P(s.Qm), Ql=dev.P(s.Ql),
            Qz=dev.P(s.Qz), Qm_inv=dev.P(s.Qm_inv), Ql_inv=dev.P(s.Ql_inv),
            Qz_inv=dev.P(s.Qz_inv), kappa=s.kappa, qz_cr=dev.P(s.qz_cr),
            row0=self.row0, row1=0 if not self.is_slab else self.row1,
            halo_u=dev.P(self.halo_u), halo_mu=dev.P(self.halo_mu), qz_w=dev.P(s.qz_w))
        if s.family == FAMILY_TRI and os.environ.get("TK_TOEPLITZ", "1") != "0" and \
                all(_toeplitz(q) for q in (s.Qm, s.Ql, s.Qz)):
            # uniform-mesh mass matrices: one scalar per weight diagonal in the row kernels
            self.level.flags |= _lib.TK_FLAG_TOEPLITZ_W
        self.lref = C.byref(self.level)
        self._fac = None
        self._scratch = None
        self._chain = None

    # --- slab geometry (local offsets of the boundary segments) -------------
    def seg_offset(self, kind: str, row: int) -> int:
        """Local offset of segment `kind` of global block row `row`."""
        nu, nz, N = self.n_u, self.n_z, self.n_steps
        start = row_start(N, nu, nz, row) - row_start(N, nu, nz, self.row0)
        if row == 0:
            off = {"u": 0, "z": nu, "lam": nu + nz}[kind]
        elif row == N:
            off = {"v": 0, "mu": nu}[kind]
        else:
            off = {"v": 0, "u": nu, "z": 2 * nu, "mu": 2 * nu + nz, "lam": 3 * nu + nz}[kind]
        return start + off

    def ensure_subst(self) -> None:
        """Precompute the Gauss-Seidel chain data once: the per-interval factor
        records (tk_subst_factor) and, for TRI levels long enough to gain from
        it, the time-chunk propagators of the coupling chain (tk_chain_prod).
        Afterwards tk_forward_subst / tk_backward_subst run as parallel solve
        -> (chunked) coupling chain -> parallel solve.  ``TK_SERIAL_SUBST=1``
        keeps the plain serial kernels (used by tests to cross-check);
        ``TK_CHAIN_CHUNK=Lc`` overrides the chunk length (0: serial chain)."""
        if os.environ.get("TK_SERIAL_SUBST") == "1":
            return
        self._ensure_fac()
        self._ensure_chain()

    def _ensure_fac(self) -> None:
        if self._fac is not None or os.environ.get("TK_SERIAL_SUBST") == "1":
            return
        lib = _lib.load()
        nf = int(lib.tk_subst_factor_len(self.lref))
        ns = int(lib.tk_subst_scratch_len(self.lref))
        self._fac = dev.empty(nf)
        self._scratch = dev.empty(ns)
        self.level.fac = self._fac.data_ptr()
        self.level.scratch = self._scratch.data_ptr()
        dev.call("tk_subst_factor", self.lref, dev.stream())
        # TRI: the records also drive every D^{-1} (Jacobi, diagonal solve)
        if os.environ.get("TK_NO_RECORDS") == "1":
            self.level.flags |= _lib.TK_FLAG_ONTHEFLY

    def _ensure_chain(self) -> None:
        if self._chain is not None or self.family != FAMILY_TRI or self.is_slab:
            return
        lib = _lib.load()
        env = os.environ.get("TK_CHAIN_CHUNK")
        lc = int(env) if env is not None else int(lib.tk_chain_chunk_default(self.n_u, self.n_steps))
        self._chain = ()
        if lc <= 0:
            return
        self.level.chain_chunk = lc
        n = int(lib.tk_chain_prod_len(self.lref))
        self._chain = dev.empty(max(n, 1))
        self.level.chain_prod = self._chain.data_ptr()
        dev.call("tk_chain_prod", self.lref, dev.stream())

    @property
    def has_records(self) -> bool:
        """Factor records present (tk_subst_factor ran), so the substitutions
        run as parallel solve -> chain -> parallel solve."""
        return self._fac is not None

    def ensure_records(self, force: bool = False) -> None:
        """TRI levels beyond the partitioned on-the-fly solve (n_u > 2048,
        or ``force``/``TK_RECORDS_ALL=1``): precompute the per-interval factor
        records once so that every local solve runs rhs-only.  Smaller levels
        refactor on the fly, which moves fewer HBM bytes per sweep."""
        if self.family != FAMILY_TRI:
            return
        if force or self.n_u > 2048 or os.environ.get("TK_RECORDS_ALL") == "1":
            self._ensure_fac()
            if force:            # the record-based row kernels even where tri_rows_part runs
                self.level.flags |= _lib.TK_FLAG_RECROWS

    @property
    def dim(self) -> int:
        return self.stage.dim

    @property
    def family(self) -> int:
        return self.stage.family

    @property
    def layout(self) -> KktLayout:
        if self._layout is None:
            self._layout = KktLayout(self.n_steps, self.n_u, self.n_z)
        return self._layout

    def _chk(self, x):
        if x.shape != (self.dim,):
            raise DimensionMismatch(f"vector shape {tuple(x.shape)} != ({self.dim},)")

    def apply(self, x, out=None):
        """y = A x (kkt.py:228)."""
        host = dev.is_host(x)
        x = dev.to_device(x)
        self._chk(x)
        y = dev.empty(self.dim) if out is None else out
        dev.call("tk_kkt_apply", self.lref, dev.P(x), dev.P(y), dev.stream())
        return dev.to_host(y) if host else y

    def residual(self, b, x, out=None):
        """r = b - A x."""
        host = dev.is_host(b)
        b, x = dev.to_device(b), dev.to_device(x)
        self._chk(b); self._chk(x)
        r = dev.empty(self.dim) if out is None else out
        dev.call("tk_kkt_residual", self.lref, dev.P(b), dev.P(x), dev.P(r), dev.stream())
        return dev.to_host(r) if host else r

    def apply_diag(self, x, out=None):
        """y = D x (block diagonal part, kkt.py:400-410)."""
        host = dev.is_host(x)
        x = dev.to_device(x)
        self._chk(x)
        y = dev.empty(self.dim) if out is None else out
        dev.call("tk_kkt_apply_diag", self.lref, dev.P(x), dev.P(y), dev.stream())
        return dev.to_host(y) if host else y

    def as_operator(self):
        from .krylov import LinearOperator
        return LinearOperator(dim=self.dim, apply=self.apply)

    def materialize(self) -> np.ndarray:
        """Dense matrix by applying A to the unit vectors (small N only)."""
        if self.dim > 6000:
            raise ValueError("materialize is meant for small desk instances")
        eye = torch.eye(self.dim, dtype=dev.F64, device=dev.device())
        cols = [self.apply(eye[j].contiguous()) for j in range(self.dim)]
        return dev.to_host(torch.stack(cols, dim=1))


def assemble_kkt(s: StageBlocks, nu: Optional[int] = None,
                 nz: Optional[int] = None) -> BlockTriKKT:
    """kkt.py:279-320 -- the operator is matrix-free over the stage data."""
    if (nu is not None and nu != s.n_u) or (nz is not None and nz != s.n_z):
        raise DimensionMismatch("stage blocks do not match the stated dimensions")
    return BlockTriKKT(s)


class DiagonalSolver:
    """D^{-1} over all block rows (kkt.py:338-389), one exact local KKT solve
    per time interval on the device (no explicit inverses are formed)."""

    def __init__(self, a: BlockTriKKT):
        self.a = a
        self.layout = a.layout if a.dim <= 1 << 22 else None
        self.n_steps = a.n_steps

    def solve_all(self, r, out=None):
        host = dev.is_host(r)
        r = dev.to_device(r)
        self.a._chk(r)
        y = dev.empty(self.a.dim) if out is None else out
        dev.call("tk_diag_solve", self.a.lref, dev.P(r), dev.P(y), dev.stream())
        return dev.to_host(y) if host else y

    def solve_block(self, i: int, r_block):
        """Solve one diagonal block (convenience; embeds it in a full vector)."""
        lay = self.a.layout
        s, w = lay.block_starts[i], lay.block_size(i)
        full = np.zeros(self.a.dim)
        full[s:s + w] = np.asarray(dev.to_host(r_block) if isinstance(r_block, torch.Tensor)
                                   else r_block)
        return dev.to_host(self.solve_all(dev.to_device(full)))[s:s + w]
