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
import functools
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import _lib
from . import device as dev
from .errors import DimensionMismatch, SingularBlock, UnsupportedStructure
from .timedisc import ProblemSpec, stage_jacobians, stage_weights

FAMILY_DENSE = _lib.FAMILY_DENSE
FAMILY_TRI = _lib.FAMILY_TRI
MAX_DENSE = 4
MAX_DENSE_GENERAL, MAX_DENSE_GENERAL_NZ = 40, 8     # warp-per-row dense kernels (tk_denseg.cu)
PIVOT_FLOOR = 1e-14            # linalg.py:38


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


def _tri_dense(d: np.ndarray) -> np.ndarray:
    """(N, 3, n) (sub, diag, sup) diagonals -> (N, n, n) dense matrices."""
    N, _, n = d.shape
    out = np.zeros((N, n, n))
    i = np.arange(n)
    out[:, i, i] = d[:, 1]
    out[:, i[1:], i[:-1]] = d[:, 0, 1:]
    out[:, i[:-1], i[1:]] = d[:, 2, :-1]
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

    # reference-layout host arrays of the stored stages (kkt.py:63-68), when the
    # stages came from host arrays; otherwise built lazily from the device data
    host_arrays: Optional[dict] = field(default=None, repr=False)
    # B_i of a TRI family built natively (reference formula, stage-constant)
    b_const: Optional[np.ndarray] = field(default=None, repr=False)

    def __post_init__(self):
        if self.n_global == 0:
            self.n_global = self.n_steps

    # --- the reference's StageBlocks fields (kkt.py:53-80), host numpy ------
    # Callers of the reference (sqp.py:252-313 apply_cx / apply_cx_t /
    # hessian_operator) read k, c, b, q_u, q_v, q_z as (N, ., .) arrays.  They
    # are materialised on first access (dense: N n_u^2 doubles each), so they
    # are meant for desk-size instances; the device path never reads them.
    def _stage_host(self, name):
        if self.host_arrays is not None:
            return self.host_arrays[name]
        return None

    @functools.cached_property
    def k(self) -> np.ndarray:
        a = self._stage_host("k")
        return a if a is not None else self._dense_stage(self.K)

    @functools.cached_property
    def c(self) -> np.ndarray:
        a = self._stage_host("c")
        return a if a is not None else self._dense_stage(self.C)

    @functools.cached_property
    def b(self) -> np.ndarray:
        a = self._stage_host("b")
        if a is not None:
            return a
        if self.family == FAMILY_DENSE:
            return dev.to_host(self.B[:self.n_steps]).copy()
        bc = self.b_const if self.b_const is not None else \
            self.kappa * self.host_weights["q_z"]
        return np.broadcast_to(bc, (self.n_steps,) + bc.shape).copy()

    def _weight_seq(self, name):
        a = self._stage_host(name)
        if a is not None:
            return a
        hw = self.host_weights
        if name == "q_z":
            return np.broadcast_to(hw["q_z"], (self.n_steps,) + hw["q_z"].shape).copy()
        out = np.broadcast_to(hw["q_mid"], (self.n_steps,) + hw["q_mid"].shape).copy()
        if self.row0 + self.n_steps >= self.n_global and self.n_steps > 0:
            out[-1] = hw["q_last"]           # the terminal stage N-1 is stored
        return out

    @functools.cached_property
    def q_u(self) -> np.ndarray:
        return self._weight_seq("q_u")

    @functools.cached_property
    def q_v(self) -> np.ndarray:
        return self._weight_seq("q_v")

    @functools.cached_property
    def q_z(self) -> np.ndarray:
        return self._weight_seq("q_z")

    def _dense_stage(self, t) -> np.ndarray:
        a = dev.to_host(t[:self.n_steps])
        if self.family == FAMILY_DENSE:
            return a.copy()
        return _tri_dense(a)

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
    if n_u <= MAX_DENSE_GENERAL and n_z <= MAX_DENSE_GENERAL_NZ:
        return FAMILY_DENSE        # general dense blocks (e.g. heat-Neumann, problems.py:218-266)
    raise UnsupportedStructure(
        f"stage blocks with n_u={n_u}, n_z={n_z} are neither dense of moderate size "
        f"(n_u <= {MAX_DENSE_GENERAL}, n_z <= {MAX_DENSE_GENERAL_NZ}) nor tridiagonal with "
        "B = kappa*Qz")


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
    # reference-built ProblemSpecs (timedisc.py:61-94) carry no `native` tag
    nat = getattr(p, "native", None)
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
        fz = p.mass      # F_z of the P1 Burgers semi-discretisation (problems.py:149-197)
        b_const = dt * p.theta * fz + dt * (1.0 - p.theta) * fz      # timedisc.py:148
        return StageBlocks(FAMILY_TRI, ns, nu, nz, K, Cm, None, **w, **slab, b_const=b_const)
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
    st = stage_blocks_from_arrays(k, c, b, qu, qu.copy(), qz)
    if rows is None:
        return st
    st.host_arrays = {nm: a[s0:max(s1, s0 + 1)] for nm, a in st.host_arrays.items()}
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
    ha = dict(k=k, c=c, b=b, q_u=q_u, q_v=q_v, q_z=q_z)
    if fam == FAMILY_DENSE:
        w = _weights(fam, q_mid, q_last, qz, 0.0)
        return StageBlocks(fam, n, nu, nz, dev.to_device(k), dev.to_device(c),
                           dev.to_device(b), **w, host_arrays=ha)
    if not all(_is_tridiagonal(a) for a in (k[i] for i in range(n))) or \
            not all(_is_tridiagonal(a) for a in (c[i] for i in range(n))):
        raise UnsupportedStructure("K_i / C_i are not tridiagonal")
    kd = np.stack([_tri_diags(k[i]) for i in range(n)])
    cd = np.stack([_tri_diags(c[i]) for i in range(n)])
    w = _weights(fam, q_mid, q_last, qz, kappa)
    return StageBlocks(fam, n, nu, nz, dev.to_device(kd), dev.to_device(cd), None, **w,
                       host_arrays=ha)


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
        if self.family == FAMILY_DENSE and (self.n_u > MAX_DENSE or self.n_z > MAX_DENSE):
            return          # general dense sizes: the substitutions run as one serial kernel
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
    per time interval on the device (no explicit inverses are formed).

    Construction verifies the blocks like the reference's factorisation
    (kkt.py:347-368): a block whose partial-pivoting LU meets a pivot below
    ``pivot_floor * max|block|`` raises :class:`SingularBlock` with its block
    index.  DENSE levels run exactly that test on every assembled block
    (tk_check_blocks); TRI blocks are symmetric quasi-definite, hence
    nonsingular, once the weights are SPD, which is what is checked there.
    """

    def __init__(self, a: BlockTriKKT, pivot_floor: float = PIVOT_FLOOR):
        self.a = a
        self.layout = a.layout if a.dim <= 1 << 22 else None
        self.n_steps = a.n_steps
        _check_blocks(a, pivot_floor)

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


# ---------------------------------------------------------------------------
# Theorem 1 verification (kkt.py:496-543) and the block singularity test
# ---------------------------------------------------------------------------
@dataclass
class Theorem1Report:
    """Per-condition, per-stage verification of the diagonal-block
    nonsingularity hypotheses (kkt.py:496-517): Q blocks SPD, K nonsingular."""

    q_u_ok: np.ndarray
    q_v_ok: np.ndarray
    q_z_ok: np.ndarray
    k_ok: np.ndarray

    @property
    def passed(self) -> bool:
        return bool(self.q_u_ok.all() and self.q_v_ok.all()
                    and self.q_z_ok.all() and self.k_ok.all())

    def failures(self):
        out = []
        for name, arr in (("q_u", self.q_u_ok), ("q_v", self.q_v_ok),
                          ("q_z", self.q_z_ok), ("k", self.k_ok)):
            for i in np.nonzero(~arr)[0]:
                out.append((name, int(i)))
        return out


def _is_spd(m: np.ndarray) -> bool:
    """Symmetric to 1e-12 relative and Cholesky-factorable (kkt.py:520-527)."""
    import scipy.linalg
    m = np.asarray(m, dtype=np.float64)
    if not np.allclose(m, m.T, rtol=0.0, atol=1e-12 * max(1.0, np.abs(m).max())):
        return False
    try:
        scipy.linalg.cholesky(m, lower=True, check_finite=False)
    except (scipy.linalg.LinAlgError, ValueError):
        return False
    return True


def _stage_flags(s: StageBlocks, pivot_floor: float) -> np.ndarray:
    """k_ok per stored stage from tk_check_k (one thread per stage on the device)."""
    ns = s.n_steps
    if ns == 0:
        return np.ones(0, dtype=bool)
    bad = torch.zeros(ns, dtype=torch.int32, device=dev.device())
    a = BlockTriKKT(s)
    dev.call("tk_check_k", a.lref, float(pivot_floor), bad.data_ptr(), dev.stream())
    return bad.cpu().numpy() == 0


def check_theorem1(s: StageBlocks, pivot_floor: float = PIVOT_FLOOR) -> Theorem1Report:
    """Report-only verification of Theorem 1's hypotheses (kkt.py:530-543).

    The weights are time-constant apart from the terminal stage, so the SPD
    tests run once per distinct weight on the host; the K_i test is the
    partial-pivoting LU pivot floor of linalg.lu_factor (linalg.py:75-103),
    evaluated per stage on the device (tk_check_k).
    """
    n = s.n_steps
    hw = s.host_weights
    if not hw:
        raise UnsupportedStructure("stage blocks carry no host copy of their weights")
    term = s.row0 + n >= s.n_global        # the terminal stage N-1 is stored here
    mid_ok, last_ok, z_ok = _is_spd(hw["q_mid"]), _is_spd(hw["q_last"]), _is_spd(hw["q_z"])
    q_ok = np.full(n, mid_ok)
    if term and n > 0:
        q_ok[-1] = last_ok
    return Theorem1Report(q_u_ok=q_ok, q_v_ok=q_ok.copy(), q_z_ok=np.full(n, z_ok),
                          k_ok=_stage_flags(s, pivot_floor))


def _check_blocks(a: BlockTriKKT, pivot_floor: float) -> None:
    """Raise SingularBlock(i) for the first diagonal block the reference's
    DiagonalSolver could not factor (kkt.py:347-368)."""
    s = a.stage
    if s.family == FAMILY_DENSE and not a.is_slab:
        bad = torch.zeros(a.n_steps + 1, dtype=torch.int32, device=dev.device())
        dev.call("tk_check_blocks", a.lref, float(pivot_floor), bad.data_ptr(), dev.stream())
        idx = np.nonzero(bad.cpu().numpy())[0]
        if idx.size:
            i = int(idx[0])
            raise SingularBlock(i, f"diagonal block {i}: pivot below floor "
                                   f"{pivot_floor:.1e} * max|block|")
        return
    hw = s.host_weights
    if s.family == FAMILY_TRI and hw:
        for name in ("q_mid", "q_last", "q_z"):
            if not _is_spd(hw[name]):
                raise UnsupportedStructure(
                    f"TRI local solves need SPD weights ({name} is not); the reference "
                    "would factor these blocks by pivoted LU")


# ---------------------------------------------------------------------------
# Splitting views, orderings, right-hand side assembly, debugging dump
# (kkt.py:323-335, 392-493, 546-560): callers of the path, host-side helpers
# ---------------------------------------------------------------------------
KINDS = ("u", "v", "z", "lam", "mu")


def factor_diagonal(a: BlockTriKKT, pivot_floor: float = PIVOT_FLOOR) -> "DiagonalSolver":
    """Verified block-diagonal solver of ``a`` (kkt.py:323-335).  The
    reference returns per-block pivoted LU factors; here the local KKT solves
    are refactored on the device at every application, so the "factors" are
    the checked :class:`DiagonalSolver` (``solve_block(i, r)`` /
    ``solve_all(r)``).  Raises :class:`SingularBlock` with the offending block
    index exactly when the reference's factorisation does."""
    return DiagonalSolver(a, pivot_floor)


def split_parts(a: BlockTriKKT):
    """Operator views (D, L, U) of A = D - L - U (kkt.py:392-425): D is the
    block diagonal (tk_kkt_apply_diag), L and U the negated strictly lower /
    upper parts, i.e. the continuity couplings (L x)_mu = -x_u, (U x)_u = -x_mu."""
    from .krylov import LinearOperator
    lay = a.layout
    iu = torch.from_numpy(lay.rows("u").reshape(-1)).to(dev.device())
    im = torch.from_numpy(lay.rows("mu").reshape(-1)).to(dev.device())

    def _wrap(fn):
        def apply(x):
            host = dev.is_host(x)
            xd = dev.to_device(x)
            a._chk(xd)
            y = fn(xd)
            return dev.to_host(y) if host else y
        return apply

    def lower_neg(x):
        y = torch.zeros_like(x)
        y[im] = -x[iu]
        return y

    def upper_neg(x):
        y = torch.zeros_like(x)
        y[iu] = -x[im]
        return y

    return (LinearOperator(dim=lay.dim, apply=_wrap(a.apply_diag)),
            LinearOperator(dim=lay.dim, apply=_wrap(lower_neg)),
            LinearOperator(dim=lay.dim, apply=_wrap(upper_neg)))


def _clustered_rows(n: int, nu: int, nz: int) -> dict:
    """Index arrays of the variable-clustered ordering (kkt.py:428-440):
    (u_t, v_t) pairs over time, then every z_t, then (lam_t, mu_t) pairs."""
    t = np.arange(n)[:, None]
    ku, kz = np.arange(nu)[None, :], np.arange(nz)[None, :]
    mult = 2 * n * nu + n * nz
    return {"u": 2 * nu * t + ku, "v": 2 * nu * t + nu + ku, "z": 2 * n * nu + nz * t + kz,
            "lam": mult + 2 * nu * t + ku, "mu": mult + 2 * nu * t + nu + ku}


def clustered_permutation(nu: int, nz: int, n: int) -> np.ndarray:
    """``perm`` with ``x_time_clustered = x_variable_clustered[perm]`` (kkt.py:443-450)."""
    lay = KktLayout(n, nu, nz)
    src = _clustered_rows(n, nu, nz)
    perm = np.empty(lay.dim, dtype=np.intp)
    for kind in KINDS:
        perm[lay.rows(kind).ravel()] = src[kind].ravel()
    return perm


def _check_len(x, nu, nz, n):
    x = np.asarray(x)
    dim = n * (4 * nu + nz)
    if x.shape != (dim,):
        raise DimensionMismatch(f"vector shape {x.shape} != ({dim},)")
    return x


def from_clustered(x_clustered, nu: int, nz: int, n: int) -> np.ndarray:
    """Variable-clustered -> time-clustered ordering (kkt.py:453-459)."""
    return _check_len(x_clustered, nu, nz, n)[clustered_permutation(nu, nz, n)]


def to_clustered(x_ordered, nu: int, nz: int, n: int) -> np.ndarray:
    """Inverse of :func:`from_clustered` (kkt.py:462-470)."""
    x = _check_len(x_ordered, nu, nz, n)
    out = np.empty_like(x)
    out[clustered_permutation(nu, nz, n)] = x
    return out


def assemble_rhs(s: StageBlocks, b1, b1v, b2, b3, b4) -> np.ndarray:
    """Right-hand side in the time-clustered ordering (kkt.py:473-493): the
    targets b1, b1v, b2 enter weighted by Q_u, Q_v, Q_z on the u, v, z rows,
    the dynamics and continuity residuals b3, b4 fill the lam and mu rows."""
    n, nu, nz = s.n_steps, s.n_u, s.n_z
    lay = KktLayout(n, nu, nz)
    rhs = np.empty(lay.dim)
    for kind, q, t, w in (("u", s.q_u, b1, nu), ("v", s.q_v, b1v, nu), ("z", s.q_z, b2, nz)):
        t = np.asarray(t, dtype=np.float64).reshape(n, w)
        rhs[lay.rows(kind)] = np.einsum("tij,tj->ti", q, t)
    rhs[lay.rows("lam")] = np.asarray(b3, dtype=np.float64).reshape(n, nu)
    rhs[lay.rows("mu")] = np.asarray(b4, dtype=np.float64).reshape(n, nu)
    return rhs


def dump_matrix_market(a: BlockTriKKT, path: str) -> None:
    """Coordinate-format text dump of the dense materialisation, for small N
    (kkt.py:546-560): MatrixMarket header, ``rows cols nnz``, 1-based entries."""
    dense = a.materialize()
    ii, jj = np.nonzero(dense)
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("%%MatrixMarket matrix coordinate real general\n")
        fh.write(f"% block-tridiagonal augmented system, N={a.n_steps} "
                 f"n_u={a.n_u} n_z={a.n_z}\n")
        fh.write(f"{dense.shape[0]} {dense.shape[1]} {ii.size}\n")
        for i, j in zip(ii, jj):
            fh.write(f"{i + 1} {j + 1} {dense[i, j]:.17g}\n")
