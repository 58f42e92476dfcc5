"""ctypes binding of libtempokkt_b200.so (the C-ABI in include/tempokkt_b200.h).

There is no fallback: if the shared library is missing or cannot be loaded
the import of any compute entry point raises :class:`NativeLibraryError`.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import NativeLibraryError, TempoKktError

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TK_LIB_PATH", os.path.join(_PKG, "libtempokkt_b200.so"))

TK_OK = 0
TK_ERR_ARG = 1
TK_ERR_CUDA = 2
TK_ERR_UNSUPPORTED = 3
TK_ERR_NEWTON = 4
FAMILY_DENSE = 0
FAMILY_TRI = 1

_p = C.c_void_p
_d = C.c_double
_i32 = C.c_int32
_i64 = C.c_int64


TK_FLAG_ONTHEFLY = 1
TK_FLAG_RECROWS = 2
TK_FLAG_TOEPLITZ_W = 4


class TkLevel(C.Structure):
    """Mirror of ``struct tk_level`` (include/tempokkt_b200.h)."""
    _fields_ = [
        ("family", _i32), ("n_steps", _i32), ("n_u", _i32), ("n_z", _i32),
        ("K", _p), ("C", _p), ("B", _p),
        ("Qm", _p), ("Ql", _p), ("Qz", _p),
        ("Qm_inv", _p), ("Ql_inv", _p), ("Qz_inv", _p),
        ("kappa", _d), ("qz_cr", _p),
        ("fac", _p), ("scratch", _p),
        ("row0", _i32), ("row1", _i32), ("halo_u", _p), ("halo_mu", _p),
        ("qz_w", _p),
        ("chain_prod", _p), ("chain_chunk", _i32), ("flags", _i32),
    ]


_SIGS = {
    "tk_version": (C.c_char_p, []),
    "tk_last_error": (C.c_char_p, []),
    "tk_kkt_dim": (_i64, [_i32, _i32, _i32]),
    "tk_tri_smem_bytes": (_i64, [_i32]),
    "tk_kkt_apply": (C.c_int, [C.POINTER(TkLevel), _p, _p, _p]),
    "tk_kkt_residual": (C.c_int, [C.POINTER(TkLevel), _p, _p, _p, _p]),
    "tk_kkt_apply_diag": (C.c_int, [C.POINTER(TkLevel), _p, _p, _p]),
    "tk_diag_solve": (C.c_int, [C.POINTER(TkLevel), _p, _p, _p]),
    "tk_jacobi_sweep": (C.c_int, [C.POINTER(TkLevel), _p, _p, _p, _d, _p]),
    "tk_jacobi0_restrict_ok": (_i32, [C.POINTER(TkLevel), _d]),
    "tk_jacobi0_restrict": (C.c_int, [C.POINTER(TkLevel), _p, _d, _p, _p, _p]),
    "tk_jacobi_prolong_ok": (_i32, [C.POINTER(TkLevel), _d]),
    "tk_jacobi_restrict": (C.c_int, [C.POINTER(TkLevel), _p, _p, _p, _p, _p]),
    "tk_jacobi0_restrict_um": (C.c_int, [C.POINTER(TkLevel), _p, _p, _p, _p]),
    "tk_jacobi_prolong": (C.c_int, [C.POINTER(TkLevel), _p, _p, _p, _p, _p]),
    "tk_restrict_fix_slab": (C.c_int, [C.POINTER(TkLevel), _p, _p]),
    "tk_restrict_fix_slab_x": (C.c_int, [C.POINTER(TkLevel), _p, _i32, _p]),
    "tk_jacobi_prolong_slab": (C.c_int, [C.POINTER(TkLevel), _p, _p, _p, _p, _p, _p]),
    "tk_forward_subst": (C.c_int, [C.POINTER(TkLevel), _p, _p, _p]),
    "tk_backward_subst": (C.c_int, [C.POINTER(TkLevel), _p, _p, _p]),
    "tk_sgs_back_half": (C.c_int, [C.POINTER(TkLevel), _p, _p, _p]),
    "tk_subst_factor_len": (_i64, [C.POINTER(TkLevel)]),
    "tk_subst_scratch_len": (_i64, [C.POINTER(TkLevel)]),
    "tk_subst_factor": (C.c_int, [C.POINTER(TkLevel), _p]),
    "tk_tri_cut_nodes": (_i32, [_i32]),
    "tk_chain_chunk_default": (_i32, [_i32, _i32]),
    "tk_chain_prod_len": (_i64, [C.POINTER(TkLevel)]),
    "tk_chain_prod": (C.c_int, [C.POINTER(TkLevel), _p]),
    "tk_tri_cut_indices": (C.c_int, [_i32, _p]),
    "tk_restrict": (C.c_int, [_i32, _i32, _i32, _p, _p, _p]),
    "tk_prolong_add": (C.c_int, [_i32, _i32, _i32, _p, _p, _p]),
    "tk_restrict_slab": (C.c_int, [_i32, _i32, _i32, _i32, _i32, _p, _p, _p]),
    "tk_prolong_add_slab": (C.c_int, [_i32, _i32, _i32, _i32, _i32, _p, _p, _p, _p, _p]),
    "tk_residual_restrict": (C.c_int, [C.POINTER(TkLevel), _p, _p, _p, _p, _p]),
    "tk_residual_restrict_jacobi0": (C.c_int, [C.POINTER(TkLevel), _p, _p, _d, _p, _p]),
    "tk_reduce_work_len": (_i64, []),
    "tk_dot": (C.c_int, [_i64, _p, _p, _p, _p, _p]),
    "tk_nrm2": (C.c_int, [_i64, _p, _p, _p, _p]),
    "tk_axpy": (C.c_int, [_i64, _d, _p, _p, _p]),
    "tk_scale_into": (C.c_int, [_i64, _d, _p, _p, _p]),
    "tk_rsub": (C.c_int, [_i64, _p, _p, _p]),
    "tk_axpy_dev": (C.c_int, [_i64, _p, _d, _p, _p, _p]),
    "tk_sqrt_div": (C.c_int, [_i64, _p, _p, _p, _p, _p]),
    "tk_gemv_t_add": (C.c_int, [_i64, _i32, _p, _i64, _p, _p, _p]),
    "tk_arnoldi_mgs": (C.c_int, [_i64, _i32, _p, _i64, _p, _p, _p, _p]),
    "tk_copy_kernel": (C.c_int, [_i64, _p, _p, _p]),
    "tk_l2_persist_reset": (C.c_int, []),
    "tk_l2_persist_allow": (C.c_int, [_i32]),
    "tk_arnoldi_supported": (_i32, []),
    "tk_graph_capture_begin": (C.c_int, [_p]),
    "tk_graph_cond_create": (C.c_int, [_p, C.POINTER(C.c_uint64)]),
    "tk_graph_while_begin": (C.c_int, [_p, _p, C.c_uint64]),
    "tk_graph_while_end": (C.c_int, [_p]),
    "tk_graph_capture_end": (C.c_int, [_p, C.POINTER(C.c_void_p)]),
    "tk_graph_launch": (C.c_int, [_p, _p]),
    "tk_graph_destroy": (C.c_int, [_p]),
    "tk_gm_state_len": (_i64, [_i32]),
    "tk_gm_begin": (C.c_int, [_i64, _p, _p, _i64, _p, _p, _i32, _d, _i32, C.c_uint64, _p, _p]),
    "tk_gm_arnoldi": (C.c_int, [_i64, _p, _i64, _p, _p, _i32, _p, _p, _p]),
    "tk_gm_givens": (C.c_int, [_p, _i32, C.c_uint64, _p]),
    "tk_gm_storez": (C.c_int, [_i64, _p, _p, _i64, _p, _i32, _p]),
    "tk_gm_combine": (C.c_int, [_i64, _p, _i64, _p, _i32, _p, _p]),
    "tk_gm_finish": (C.c_int, [_i64, _p, _p, _p, _p, _i32, _p, _p, _p]),
    "tk_host_device_ptr": (C.c_int, [_p, C.POINTER(C.c_void_p)]),
    "tk_host_alloc_mapped": (C.c_int, [_i64, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]),
    "tk_host_free": (C.c_int, [_p]),
    "tk_stage_vanderpol": (C.c_int, [_i32, _d, _d, _d, _i32, _p, _p, _p, _p, _p, _p, _p, _p]),
    "tk_stage_burgers": (C.c_int, [_i32, _i32, _d, _d, _d, _p, _p, _p, _p, _p, _p]),
    "tk_forward_vanderpol_host": (C.c_int, [_i32, _d, _d, _d, _i32, _p, _p, _d, _p]),
    "tk_forward_burgers_host": (C.c_int, [_i32, _i32, _d, _d, _d, _p, _p, _d, _p]),
    "tk_check_k": (C.c_int, [C.POINTER(TkLevel), _d, _p, _p]),
    "tk_check_blocks": (C.c_int, [C.POINTER(TkLevel), _d, _p, _p]),
    "tk_cr_scalar_factor": (C.c_int, [_i32, _p, _p]),
    "tk_cr_scalar_solve_host": (C.c_int, [_i32, _p, _p, _p]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load(path: str = LIB_PATH):
    """Load (once) and type the shared library; raise loudly if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeLibraryError(
            f"{path} not found: build it with `python -m paper_2405_04808_b200.build` "
            "(there is no CPU fallback for the hot path)")
    try:
        lib = C.CDLL(path)
    except OSError as exc:  # pragma: no cover - environment specific
        raise NativeLibraryError(f"cannot load {path}: {exc}") from exc
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int, what: str = "") -> None:
    if rc != TK_OK:
        msg = load().tk_last_error().decode(errors="replace")
        raise TempoKktError(f"{what or 'tempokkt_b200'} failed (code {rc}): {msg}")


def ptr(t) -> int:
    """Raw device/host pointer of a torch tensor or numpy array (or None)."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    return t.ctypes.data
