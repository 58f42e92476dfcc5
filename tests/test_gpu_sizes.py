"""GPU vs oracle at spatial sizes that exercise every cyclic-reduction path:
several CTA-wide and warp levels, the dense cut solve with more rows than
threads, non-power-of-two n, and both the on-the-fly and the record-based
local solves."""

import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu


def _case(n_u, n=16, theta=0.5, seed=0):
    import paper_2405_04808_b200 as P
    from oracle import tk_oracle as O
    grid = P.TimeGrid(1.0, n)
    p = P.build_burgers(P.BurgersConfig(n_elems=n_u + 1, theta=theta, u0_kind="sinstep"), grid)
    op = O.burgers(n_u=n_u, nu=1e-2, alpha=0.1, theta=theta, u0_kind="sinstep")
    rng = np.random.default_rng(seed)
    u = P.forward_solve(p, np.zeros((n, n_u)), grid).states
    v = u + 0.01 * rng.standard_normal(u.shape)
    z = 0.1 * rng.standard_normal((n, n_u))
    return P, O, p, op, grid, u, v, z, rng


@pytest.mark.parametrize("n_u", [33, 64, 100, 128, 256, 300, 512])
@pytest.mark.parametrize("records", [False, True])
def test_operator_and_smoothers(n_u, records):
    P, O, p, op, grid, u, v, z, rng = _case(n_u)
    st = P.build_stage_blocks(p, grid.dt, u, v, z)
    a = P.assemble_kkt(st)
    if records:
        a.ensure_records(force=True)
    ost = O.build_stages(op, grid.dt, u, v, z)
    oa = O.Kkt(ost)
    od = O.DiagSolve(oa)
    x = rng.standard_normal(a.dim)
    b = rng.standard_normal(a.dim)
    assert rel(a.apply(x), oa.apply(x)) < 1e-13
    assert rel(P.DiagonalSolver(a).solve_all(b), od.all(b)) < 1e-11
    assert rel(P.jacobi_apply(a, None, b, x, 2), O.jacobi(oa, od, b, x, 2)) < 1e-11
    assert rel(P.fgs_apply(a, None, b, x), O.fgs(oa, od, b, x)) < 1e-11
    assert rel(P.bgs_apply(a, None, b, x), O.bgs(oa, od, b, x)) < 1e-11
    assert rel(P.sgs_apply(a, None, b, x), O.sgs(oa, od, b, x)) < 1e-11


@pytest.mark.parametrize("n_u", [64, 128])
def test_cycle_and_solve(n_u):
    P, O, p, op, grid, u, v, z, rng = _case(n_u, n=32)
    h = P.build_hierarchy(p, u, v, z, grid, 3, sweeps=1, coarse_tol=1e-2)
    oh = O.build_hierarchy(op, u, v, z, 32, grid.dt, 3, sweeps=1, coarse_tol=1e-2)
    b = rng.standard_normal(h.levels[0].kkt.dim)
    assert rel(P.cycle(h, 0, b), O.cycle(oh, 0, b)) < 1e-10
    assert h.stats.iters == oh.coarse_iters
    h.stats = type(h.stats)()
    oh.coarse_iters = oh.coarse_calls = 0
    x, rep = P.fgmres(h.levels[0].kkt.as_operator(), P.mg_preconditioner(h), b, rel_tol=1e-8,
                      max_iters=60)
    xo, orep = O.fgmres(oh.levels[0].kkt.apply, O.mg_prec(oh), b, rel_tol=1e-8, max_iters=60)
    assert rep.iterations == orep.iterations
    assert h.stats.iters == oh.coarse_iters
    assert rel(x, xo) < 1e-10


@pytest.mark.parametrize("lc", [1, 3, 4, 7, 31, 62, 63, 100])
def test_chunked_chain(lc, monkeypatch):
    """Time-chunked coupling chain (zero-start chunks -> carry with the chunk
    propagators -> re-run) against the oracle's serial substitutions, for
    chunk lengths giving one, two, and many chunks and a ragged last chunk."""
    monkeypatch.setenv("TK_CHAIN_CHUNK", str(lc))
    P, O, p, op, grid, u, v, z, rng = _case(64, n=64)
    st = P.build_stage_blocks(p, grid.dt, u, v, z)
    a = P.assemble_kkt(st)
    a.ensure_subst()
    assert a.level.chain_chunk == lc
    oa = O.Kkt(O.build_stages(op, grid.dt, u, v, z))
    od = O.DiagSolve(oa)
    x = rng.standard_normal(a.dim)
    b = rng.standard_normal(a.dim)
    assert rel(P.fgs_apply(a, None, b, x), O.fgs(oa, od, b, x)) < 1e-11
    assert rel(P.bgs_apply(a, None, b, x), O.bgs(oa, od, b, x)) < 1e-11
    assert rel(P.sgs_apply(a, None, b, x), O.sgs(oa, od, b, x)) < 1e-11


def test_chunked_coarse_cycle():
    """Default chunking on a 64-interval coarse level inside a V-cycle and
    the preconditioned FGMRES: same coarse and outer iteration counts."""
    P, O, p, op, grid, u, v, z, rng = _case(64, n=128)
    h = P.build_hierarchy(p, u, v, z, grid, 2, sweeps=1, coarse_tol=1e-2)
    assert h.levels[-1].kkt.level.chain_chunk > 0
    oh = O.build_hierarchy(op, u, v, z, 128, grid.dt, 2, sweeps=1, coarse_tol=1e-2)
    b = rng.standard_normal(h.levels[0].kkt.dim)
    assert rel(P.cycle(h, 0, b), O.cycle(oh, 0, b)) < 1e-10
    assert h.stats.iters == oh.coarse_iters
    h.stats = type(h.stats)()
    oh.coarse_iters = oh.coarse_calls = 0
    x, rep = P.fgmres(h.levels[0].kkt.as_operator(), P.mg_preconditioner(h), b, rel_tol=1e-8,
                      max_iters=40)
    xo, orep = O.fgmres(oh.levels[0].kkt.apply, O.mg_prec(oh), b, rel_tol=1e-8, max_iters=40)
    assert rep.iterations == orep.iterations
    assert h.stats.iters == oh.coarse_iters
    assert rel(x, xo) < 1e-10


@pytest.mark.parametrize("n_u", [1000, 1024, 1100, 1536, 2048])
def test_large_n_identities(n_u):
    """Large spatial sizes (BASELINE configs[4] has n_u = 2048), where dense
    oracle inverses are out of reach: the block-diagonal solve and the Jacobi
    sweep are checked through the identities D (D^{-1} b) = b and
    D (y - x) = b - A x with the (independently parity-tested) operator
    kernels."""
    import torch
    P, O, p, op, grid, u, v, z, rng = _case(n_u, n=8)
    st = P.build_stage_blocks(p, grid.dt, u, v, z)
    a = P.assemble_kkt(st)
    a.ensure_records()      # as build_hierarchy does (records for n_u > 1664)
    b = torch.from_numpy(rng.standard_normal(a.dim)).cuda()
    x = torch.from_numpy(rng.standard_normal(a.dim)).cuda()
    d = P.DiagonalSolver(a).solve_all(b)
    assert rel(a.apply_diag(d).cpu().numpy(), b.cpu().numpy()) < 1e-11
    y = P.jacobi_apply(a, None, b, x, 1)
    r = a.residual(b, x)
    assert rel(a.apply_diag(y - x).cpu().numpy(), r.cpu().numpy()) < 1e-11


@pytest.mark.parametrize("n_u", [33, 64, 100, 128, 300, 512, 1536])
@pytest.mark.parametrize("n", [16, 64])
def test_fused_jacobi0_restrict_bitwise(n_u, n):
    """tk_jacobi0_restrict == zero-start tk_jacobi_sweep + tk_residual_restrict_jacobi0,
    bit for bit (output and restricted residual), and against the oracle's
    restricted residual of that sweep."""
    import torch
    from paper_2405_04808_b200 import device as dev
    from paper_2405_04808_b200.multigrid import fused_jacobi0_ok
    from paper_2405_04808_b200.smoothers import jacobi_sweeps
    P, O, p, op, grid, u, v, z, rng = _case(n_u, n=n)
    st = P.build_stage_blocks(p, grid.dt, u, v, z)
    a = P.assemble_kkt(st)
    assert fused_jacobi0_ok(a, 1.0) and not fused_jacobi0_ok(a, 0.8)
    cdim = (n // 2) * 5 * n_u
    b = dev.to_device(rng.standard_normal(a.dim))
    x = dev.empty(a.dim)
    rc = dev.to_device(np.full(cdim, np.nan))
    dev.call("tk_jacobi0_restrict", a.lref, dev.P(b), 1.0, dev.P(x), dev.P(rc), dev.stream())
    x2 = jacobi_sweeps(a, b, None, 1, 1.0)
    rc2 = dev.empty(cdim)
    dev.call("tk_residual_restrict_jacobi0", a.lref, dev.P(b), dev.P(x2), 1.0, dev.P(rc2),
             dev.stream())
    torch.cuda.synchronize()
    assert torch.equal(x, x2)
    assert torch.equal(rc, rc2)
    ost = O.build_stages(op, grid.dt, u, v, z)
    oa = O.Kkt(ost)
    bh, xh = b.cpu().numpy(), x.cpu().numpy()
    ro = O.restrict_kkt(O.Layout(n, n_u, n_u), O.Layout(n // 2, n_u, n_u), bh - oa.apply(xh))
    assert rel(rc.cpu().numpy(), ro) < 1e-10


@pytest.mark.parametrize("n_controls", [1, 2])
def test_fused_jacobi0_restrict_dense_bitwise(n_controls):
    """DENSE (van der Pol) tk_jacobi0_restrict == zero-start sweep + restriction."""
    import torch
    import paper_2405_04808_b200 as P
    from paper_2405_04808_b200 import device as dev
    from paper_2405_04808_b200.multigrid import fused_jacobi0_ok
    from paper_2405_04808_b200.smoothers import jacobi_sweeps
    n = 64
    grid = P.TimeGrid(5.0, n)
    vp = P.build_vanderpol(P.VanDerPolConfig(n_controls=n_controls, u_init=(1.0, 0.0)), grid,
                           with_targets=False)
    rng = np.random.default_rng(4)
    zc = 0.3 * rng.standard_normal((n, n_controls))
    uv = P.forward_solve(vp, zc, grid).states
    a = P.assemble_kkt(P.build_stage_blocks(vp, grid.dt, uv, uv, zc))
    assert fused_jacobi0_ok(a, 1.0)
    cdim = (n // 2) * (4 * 2 + n_controls)
    b = dev.to_device(rng.standard_normal(a.dim))
    x = dev.empty(a.dim)
    rc = dev.to_device(np.full(cdim, np.nan))
    dev.call("tk_jacobi0_restrict", a.lref, dev.P(b), 1.0, dev.P(x), dev.P(rc), dev.stream())
    x2 = jacobi_sweeps(a, b, None, 1, 1.0)
    rc2 = dev.empty(cdim)
    dev.call("tk_residual_restrict_jacobi0", a.lref, dev.P(b), dev.P(x2), 1.0, dev.P(rc2),
             dev.stream())
    torch.cuda.synchronize()
    assert torch.equal(x, x2)
    assert torch.equal(rc, rc2)


@pytest.mark.parametrize("n_u", [64, 128, 512, 1024, 1536])
def test_toeplitz_weights_bitwise(n_u):
    """TK_FLAG_TOEPLITZ_W (scalar weight diagonals in the partitioned row
    kernels) gives the same sweeps / solves / fused pre-smoothing as the
    per-node weight loads (same values; the compiler may contract the
    products into FMAs differently, so agreement is to rounding, 1e-14); the
    uniform Burgers mesh sets the flag."""
    import torch
    from paper_2405_04808_b200 import _lib, device as dev
    from paper_2405_04808_b200.smoothers import jacobi_sweeps
    P, O, p, op, grid, u, v, z, rng = _case(n_u, n=16)
    st = P.build_stage_blocks(p, grid.dt, u, v, z)
    a = P.assemble_kkt(st)
    assert a.level.flags & _lib.TK_FLAG_TOEPLITZ_W
    b = dev.to_device(rng.standard_normal(a.dim))
    x = dev.to_device(rng.standard_normal(a.dim))
    rc = dev.empty((16 // 2) * 5 * n_u)

    def run():
        y1 = jacobi_sweeps(a, b, x, 1, 1.0)
        y2 = P.DiagonalSolver(a).solve_all(b)
        y3 = dev.empty(a.dim)
        dev.call("tk_jacobi0_restrict", a.lref, dev.P(b), 1.0, dev.P(y3), dev.P(rc), dev.stream())
        torch.cuda.synchronize()
        return y1.clone(), y2.clone(), y3.clone(), rc.clone()

    t = run()
    a.level.flags &= ~_lib.TK_FLAG_TOEPLITZ_W
    g = run()
    for p_, q_ in zip(t, g):
        assert rel(p_.cpu().numpy(), q_.cpu().numpy()) < 1e-14


@pytest.mark.parametrize("n_u", [600, 1024, 2048])
def test_large_n_substitutions_identities(n_u):
    """n_u > 512: the coupling chain streams its per-interval partition
    factors (tri_chainw_stream).  Dense oracle inverses are out of reach, so
    the block Gauss-Seidel substitutions are checked through their defining
    identities (D - L) d = r, (D - U) d = r and P_sgs d = r with the
    (independently parity-tested) operator kernels (reference
    smoothers.py:79-152, kkt.py:392-425)."""
    import torch
    from paper_2405_04808_b200.smoothers import backward_subst, forward_subst, sgs_zero
    P, O, p, op, grid, u, v, z, rng = _case(n_u, n=48)
    a = P.assemble_kkt(P.build_stage_blocks(p, grid.dt, u, v, z))
    a.ensure_subst()
    assert a.level.chain_chunk > 0                       # time-chunked chain
    d, low, up = P.split_parts(a)
    r = torch.from_numpy(rng.standard_normal(a.dim)).cuda()
    nr = float(torch.linalg.norm(r))
    f = forward_subst(a, r)
    assert float(torch.linalg.norm(d(f) - low(f) - r)) < 1e-9 * nr
    bk = backward_subst(a, r)
    assert float(torch.linalg.norm(d(bk) - up(bk) - r)) < 1e-9 * nr
    # P_sgs = (D - L) D^{-1} (D - U):  s = P_sgs^{-1} r  =>  (D - L) D^{-1} (D - U) s = r
    s = sgs_zero(a, r)
    t = d(s) - up(s)
    t = P.DiagonalSolver(a).solve_all(t)
    assert float(torch.linalg.norm(d(t) - low(t) - r)) < 1e-8 * nr


def test_grouped_carry_register_rows_identities():
    """n_u = 512 with a long level (256 intervals: 32 chunks, grouped two-level
    carry): the carry runs with one propagator row per warp in registers and
    phases B + C in one launch (tri_chain_carry_seg<FWD, RG>, mode 3) -- the
    configs[2] coarse-level path.  Checked through the substitutions' defining
    identities (reference smoothers.py:79-152), as test_large_n_substitutions_identities."""
    import torch
    from paper_2405_04808_b200.smoothers import backward_subst, forward_subst, sgs_zero
    P, O, p, op, grid, u, v, z, rng = _case(512, n=256)
    a = P.assemble_kkt(P.build_stage_blocks(p, grid.dt, u, v, z))
    a.ensure_subst()
    lc = a.level.chain_chunk
    assert lc > 0 and (255 + lc - 1) // lc - 2 > 12      # enough chunks for the grouped carry
    d, low, up = P.split_parts(a)
    r = torch.from_numpy(rng.standard_normal(a.dim)).cuda()
    nr = float(torch.linalg.norm(r))
    f = forward_subst(a, r)
    assert float(torch.linalg.norm(d(f) - low(f) - r)) < 1e-9 * nr
    bk = backward_subst(a, r)
    assert float(torch.linalg.norm(d(bk) - up(bk) - r)) < 1e-9 * nr
    s = sgs_zero(a, r)
    t = d(s) - up(s)
    t = P.DiagonalSolver(a).solve_all(t)
    assert float(torch.linalg.norm(d(t) - low(t) - r)) < 1e-8 * nr
