"""CPU tests of the C-ABI boundary: the library loads, exports every symbol
declared in include/tempokkt_b200.h, and its host routines (forward march,
scalar cyclic-reduction factor) agree with the reference's golden vectors."""

import os
import re

import numpy as np
import pytest

from conftest import ROOT, load_golden, product_problem, rel, CASES


def header_symbols():
    src = open(os.path.join(ROOT, "include", "tempokkt_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|int32_t|int64_t|const char\*)\s+(tk_\w+)\s*\(", src, re.M)))


def test_library_exports_header():
    from paper_2405_04808_b200 import _lib
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.EXPORTED)
    assert lib.tk_version().startswith(b"tempokkt_b200")
    assert lib.tk_kkt_dim(7, 2, 1) == 7 * 9


def test_null_args_rejected_without_gpu():
    from paper_2405_04808_b200 import _lib
    lib = _lib.load()
    assert lib.tk_kkt_apply(None, None, None, None) == _lib.TK_ERR_ARG
    assert lib.tk_restrict(3, 2, 1, None, None, None) == _lib.TK_ERR_ARG
    assert b"n_fine" in lib.tk_last_error() or lib.tk_last_error()
    # the fused sweeps and their time-slab versions reject null vectors before any launch
    assert lib.tk_jacobi_restrict(None, None, None, None, None, None) == _lib.TK_ERR_ARG
    assert lib.tk_jacobi_prolong_slab(None, None, None, None, None, None, None) == _lib.TK_ERR_ARG
    assert lib.tk_restrict_fix_slab(None, None, None) == _lib.TK_ERR_ARG


@pytest.mark.parametrize("name", CASES)
def test_host_forward_march_matches_reference(name):
    import paper_2405_04808_b200 as P
    g = load_golden(name)
    p, grid = product_problem(g)
    z = g["z"] if name.startswith("cfg") else np.zeros((grid.n_steps, p.n_z))
    tr = P.forward_solve(p, z, grid)
    assert rel(tr.states, g["fwd_states"]) < 1e-14


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 31, 64, 100, 513])
def test_cr_scalar_factor(n):
    from paper_2405_04808_b200 import _lib
    lib = _lib.load()
    rng = np.random.default_rng(n)
    d = 4.0 + rng.random(n)
    e = rng.random(n)
    e[-1] = 0.0
    a = np.diag(d) + np.diag(e[:-1], 1) + np.diag(e[:-1], -1)
    tri = np.zeros((3, n)); tri[1] = d; tri[2, :-1] = e[:-1]; tri[0, 1:] = e[:-1]
    coef = np.empty((3, n))
    assert lib.tk_cr_scalar_factor(n, tri.ctypes.data, coef.ctypes.data) == 0
    f = rng.standard_normal(n)
    x = np.empty(n)
    assert lib.tk_cr_scalar_solve_host(n, coef.ctypes.data, f.ctypes.data, x.ctypes.data) == 0
    assert np.abs(a @ x - f).max() < 1e-13


def test_configs_match_baseline_shapes():
    from paper_2405_04808_b200 import configs
    s = configs.build_setup(0)
    assert (s.grid.n_steps, s.n_u, s.n_z, s.levels) == (512, 2, 1, 3)
    g = load_golden("cfg0_vdp")
    assert rel(s.u, g["fwd_states"]) < 1e-14
    assert np.array_equal(s.rhs(), np.random.default_rng(0).standard_normal(512 * 9))
    s1 = configs.build_setup(1, nt=64, nx=16)
    g1 = load_golden("cfg1_burgers")
    assert rel(s1.u, g1["fwd_states"]) < 1e-14


def test_chain_sizing_without_gpu():
    """Host-side sizing of the time-chunked coupling chain (no device work):
    chunk length defaults, at most one chunk per SM, and the propagator
    buffer length including the two-level carry's group propagators."""
    from paper_2405_04808_b200 import _lib
    lib = _lib.load()
    # configs[2] coarsest level: n_u = 512, 512 intervals -> grouped carry, Lc = 12
    assert lib.tk_chain_chunk_default(512, 512) == 12
    assert lib.tk_chain_chunk_default(64, 16) == 0                 # too short to chunk
    for n_u, N in [(64, 64), (128, 128), (512, 512), (512, 4096), (2048, 512)]:
        lc = lib.tk_chain_chunk_default(n_u, N)
        assert lc >= 4 and (N - 1 + lc - 1) // lc <= 148
    lv = _lib.TkLevel(family=_lib.FAMILY_TRI, n_steps=512, n_u=512, n_z=512)
    for f in ("K", "C", "Qm", "Ql", "Qz", "qz_cr"):   # never dereferenced by the sizing
        setattr(lv, f, 16)
    lv.chain_chunk = 12
    nc = (511 + 11) // 12                                           # 43 chunks
    ng = (nc - 2 + 6 - 1) // 6                                      # groups of 6 -> 7
    n = 512
    want = 2 * nc * n * n + 3 * nc * n + 4 + 2 * ng * n * n + 2 * ng * n
    # + the warp-chain records (tk_tri_chainw.cu): n_u = 512 runs 64 threads of 8 nodes,
    # 200 coefficient slots per thread, one record per interval (16-byte aligned)
    recs = 512 * 200 * 64
    import ctypes
    assert lib.tk_chain_prod_len(ctypes.byref(lv)) == want + (want & 1) + recs
    lv.chain_chunk = 100                                            # 6 chunks: single carry
    nc = (511 + 99) // 100
    want = 2 * nc * n * n + 3 * nc * n + 4
    assert lib.tk_chain_prod_len(ctypes.byref(lv)) == want + (want & 1) + recs
