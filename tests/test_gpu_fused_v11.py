"""V(1,1), omega = 1: the splitting-form Jacobi sweep (D^{-1}(b + (L+U) x),
reference smoothers.py:61-76 with omega = 1), the pre-smoothing that stores
only the u / mu segments (tk_jacobi0_restrict_um) and the prolongation folded
into the post-smoothing sweep (tk_jacobi_prolong; reference multigrid.py:
115-132, :297-299) against the unfused kernels and the oracle."""

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


@pytest.mark.parametrize("n_u", [100, 128, 512])
def test_splitting_form_matches_residual_form_and_oracle(n_u):
    """omega = 1 sweeps (splitting form) vs the oracle's x + D^{-1}(b - A x);
    omega != 1 keeps the residual form."""
    P, O, p, op, grid, u, v, z, rng = _case(n_u)
    a = P.assemble_kkt(P.build_stage_blocks(p, grid.dt, u, v, z))
    oa = O.Kkt(O.build_stages(op, grid.dt, u, v, z))
    od = O.DiagSolve(oa)
    x = rng.standard_normal(a.dim)
    b = rng.standard_normal(a.dim)
    assert rel(P.jacobi_apply(a, None, b, x, 1, 1.0), O.jacobi(oa, od, b, x, 1, 1.0)) < 1e-11
    assert rel(P.jacobi_apply(a, None, b, x, 3, 1.0), O.jacobi(oa, od, b, x, 3, 1.0)) < 1e-11
    assert rel(P.jacobi_apply(a, None, b, x, 2, 0.7), O.jacobi(oa, od, b, x, 2, 0.7)) < 1e-11


@pytest.mark.parametrize("n_u", [33, 100, 128, 256, 300, 512, 1024, 1100, 2048])
def test_fused_pre_and_post_vs_unfused(n_u):
    import torch
    from paper_2405_04808_b200 import _lib, device as dev
    from paper_2405_04808_b200.multigrid import TransferOps
    from paper_2405_04808_b200.smoothers import jacobi_sweeps
    N = 8
    P, O, p, op, grid, u, v, z, rng = _case(n_u, n=N)
    a = P.assemble_kkt(P.build_stage_blocks(p, grid.dt, u, v, z))
    assert _lib.load().tk_jacobi_prolong_ok(a.lref, 1.0)
    t = TransferOps(N, N // 2, n_u, n_u)
    b = dev.to_device(rng.standard_normal(a.dim))
    ec = dev.to_device(rng.standard_normal(t.coarse_dim))
    # pre-smoothing: u / mu segments and rc bitwise equal, the rest untouched
    x_full, rc_full = dev.empty(a.dim), dev.empty(t.coarse_dim)
    dev.call("tk_jacobi0_restrict", a.lref, dev.P(b), 1.0, dev.P(x_full), dev.P(rc_full),
             dev.stream())
    x_um = torch.full((a.dim,), float("nan"), dtype=torch.float64, device="cuda")
    rc_um = dev.empty(t.coarse_dim)
    dev.call("tk_jacobi0_restrict_um", a.lref, dev.P(b), dev.P(x_um), dev.P(rc_um), dev.stream())
    assert torch.equal(rc_um, rc_full)
    lf, lc = O.Layout(N, n_u, n_u), O.Layout(N // 2, n_u, n_u)
    xf, xu = x_full.cpu().numpy(), x_um.cpu().numpy()
    written = np.zeros(a.dim, dtype=bool)
    written[lf.rows["u"].ravel()] = True
    written[lf.rows["mu"].ravel()] = True
    assert np.array_equal(xu[written], xf[written])
    assert np.all(np.isnan(xu[~written]))
    # post-smoothing with the prolongation inside vs tk_prolong_add + tk_jacobi_sweep
    y = dev.empty(a.dim)
    dev.call("tk_jacobi_prolong", a.lref, dev.P(b), dev.P(x_um), dev.P(ec), dev.P(y), dev.stream())
    xp = x_full.clone()
    t.prolong_add(ec, xp)
    y_ref = jacobi_sweeps(a, b, xp, 1, 1.0)
    assert rel(y.cpu().numpy(), y_ref.cpu().numpy()) < 1e-13
    if n_u <= 512:   # and against the oracle's prolongation + residual-form sweep
        oa = O.Kkt(O.build_stages(op, grid.dt, u, v, z))
        od = O.DiagSolve(oa)
        xo = xf + O.prolong_kkt(lf, lc, ec.cpu().numpy())
        assert rel(y.cpu().numpy(), O.jacobi(oa, od, b.cpu().numpy(), xo, 1, 1.0)) < 1e-11


@pytest.mark.parametrize("n_u,levels", [(100, 3), (128, 3), (256, 2)])
def test_fused_cycle_vs_oracle_and_unfused(n_u, levels, monkeypatch):
    from paper_2405_04808_b200 import multigrid as M
    P, O, p, op, grid, u, v, z, rng = _case(n_u, n=32)
    h = P.build_hierarchy(p, u, v, z, grid, levels, sweeps=1, coarse_tol=1e-2)
    assert M.fused_v11_ok(h, h.levels[0].kkt)
    oh = O.build_hierarchy(op, u, v, z, 32, grid.dt, levels, sweeps=1, coarse_tol=1e-2)
    b = rng.standard_normal(h.levels[0].kkt.dim)
    xo = O.cycle(oh, 0, b)
    x_eager = P.cycle(h, 0, b)               # first cycle: eager
    its = h.stats.iters
    assert rel(x_eager, xo) < 1e-10
    assert its == oh.coarse_iters
    x_graph = P.cycle(h, 0, b)               # second: graph replay
    assert rel(x_graph, xo) < 1e-10
    monkeypatch.setattr(M, "FUSED_PROLONG", False)
    h2 = P.build_hierarchy(p, u, v, z, grid, levels, sweeps=1, coarse_tol=1e-2)
    x_unf = P.cycle(h2, 0, b)
    assert rel(x_eager, x_unf) < 1e-12
    assert h2.stats.iters == its


@pytest.mark.parametrize("kind", ["w", "f"])
def test_fused_levels_inside_w_and_f_cycles(kind):
    """W / F cycles (multigrid.py:290-296) revisit a level with a non-zero
    iterate: only the visits from zero take the fused pair, the others the
    general kernels; both against the oracle."""
    from paper_2405_04808_b200 import multigrid as M
    P, O, p, op, grid, u, v, z, rng = _case(128, n=32)
    h = P.build_hierarchy(p, u, v, z, grid, 3, sweeps=1, coarse_tol=1e-2, cycle_kind=kind)
    assert M.fused_v11_ok(h, h.levels[0].kkt)
    oh = O.build_hierarchy(op, u, v, z, 32, grid.dt, 3, sweeps=1, coarse_tol=1e-2, cycle_kind=kind)
    b = rng.standard_normal(h.levels[0].kkt.dim)
    assert rel(P.cycle(h, 0, b), O.cycle(oh, 0, b)) < 1e-10
    assert h.stats.iters == oh.coarse_iters


@pytest.mark.parametrize("n_controls", [1, 2])
def test_dense_fused_cycle_vs_oracle_and_unfused(n_controls, monkeypatch):
    """van der Pol (DENSE family): the splitting-form rows with the folded
    prolongation (dense_rows_split) against the oracle and the unfused kernels."""
    import paper_2405_04808_b200 as P
    from oracle import tk_oracle as O
    from paper_2405_04808_b200 import multigrid as M
    n = 64
    grid = P.TimeGrid(5.0, n)
    vp = P.build_vanderpol(P.VanDerPolConfig(n_controls=n_controls, u_init=(1.0, 0.0)), grid,
                           with_targets=False)
    rng = np.random.default_rng(3)
    zc = 0.3 * rng.standard_normal((n, n_controls))
    uv = P.forward_solve(vp, zc, grid).states
    vv = uv + 0.01 * rng.standard_normal(uv.shape)
    h = P.build_hierarchy(vp, uv, vv, zc, grid, 4, sweeps=1)
    assert M.fused_v11_ok(h, h.levels[0].kkt)
    ov = O.vanderpol(n_controls=n_controls, u0=(1.0, 0.0))
    oh = O.build_hierarchy(ov, uv, vv, zc, n, grid.dt, 4, sweeps=1)
    b = rng.standard_normal(h.levels[0].kkt.dim)
    xo = O.cycle(oh, 0, b)
    x_eager = P.cycle(h, 0, b)
    assert rel(x_eager, xo) < 1e-10
    assert h.stats.iters == oh.coarse_iters
    assert rel(P.cycle(h, 0, b), xo) < 1e-10           # graph replay
    x = rng.standard_normal(h.levels[0].kkt.dim)
    a, oa = h.levels[0].kkt, oh.levels[0].kkt
    assert rel(P.jacobi_apply(a, None, b, x, 2, 1.0), O.jacobi(oa, O.DiagSolve(oa), b, x, 2, 1.0)) < 1e-11
    monkeypatch.setattr(M, "FUSED_PROLONG", False)
    h2 = P.build_hierarchy(vp, uv, vv, zc, grid, 4, sweeps=1)
    assert rel(P.cycle(h2, 0, b), x_eager) < 1e-12


@pytest.mark.parametrize("n_u", [33, 128, 300, 512, 2048])
def test_jacobi_restrict_from_nonzero_start(n_u):
    """tk_jacobi_restrict: an omega = 1 sweep from any x that also writes
    R (b - A y) = R (L + U)(y - x) (multigrid.py:285-288, last pre-smoothing
    sweep) against tk_jacobi_sweep + the general tk_residual_restrict."""
    import torch
    from paper_2405_04808_b200 import device as dev
    from paper_2405_04808_b200.multigrid import TransferOps
    from paper_2405_04808_b200.smoothers import jacobi_sweeps
    N = 8
    P, O, p, op, grid, u, v, z, rng = _case(n_u, n=N)
    a = P.assemble_kkt(P.build_stage_blocks(p, grid.dt, u, v, z))
    t = TransferOps(N, N // 2, n_u, n_u)
    b = dev.to_device(rng.standard_normal(a.dim))
    x = dev.to_device(rng.standard_normal(a.dim))
    y, rc = dev.empty(a.dim), dev.empty(t.coarse_dim)
    dev.call("tk_jacobi_restrict", a.lref, dev.P(b), dev.P(x), dev.P(y), dev.P(rc), dev.stream())
    y_ref = jacobi_sweeps(a, b, x, 1, 1.0)
    assert torch.equal(y, y_ref)
    rc_ref, work = dev.empty(t.coarse_dim), dev.empty(a.dim)
    dev.call("tk_residual_restrict", a.lref, dev.P(b), dev.P(y_ref), dev.P(rc_ref), dev.P(work),
             dev.stream())
    # b - A y cancels to rounding where the fused form writes exact zeros
    scale = float(torch.linalg.norm(b))
    assert float(torch.linalg.norm(rc - rc_ref)) < 1e-12 * scale
    # from zero (NULL): the zero-start kernel
    y0, rc0, y1, rc1 = (dev.empty(a.dim), dev.empty(t.coarse_dim), dev.empty(a.dim),
                        dev.empty(t.coarse_dim))
    dev.call("tk_jacobi_restrict", a.lref, dev.P(b), dev.P(None), dev.P(y0), dev.P(rc0), dev.stream())
    dev.call("tk_jacobi0_restrict", a.lref, dev.P(b), 1.0, dev.P(y1), dev.P(rc1), dev.stream())
    assert torch.equal(y0, y1) and torch.equal(rc0, rc1)


@pytest.mark.parametrize("kind,sweeps", [("v", 2), ("v", 3), ("w", 2), ("f", 1)])
def test_multi_sweep_fused_cycle_vs_oracle(kind, sweeps, monkeypatch):
    """sweeps > 1 and the W / F revisits with a non-zero iterate take
    tk_jacobi_restrict + tk_jacobi_prolong (eager and graph replay) --
    against the oracle and the unfused kernels."""
    from paper_2405_04808_b200 import multigrid as M
    P, O, p, op, grid, u, v, z, rng = _case(128, n=32)
    h = P.build_hierarchy(p, u, v, z, grid, 3, sweeps=sweeps, coarse_tol=1e-2, cycle_kind=kind)
    assert M.fused_vnn_ok(h, h.levels[0].kkt)
    oh = O.build_hierarchy(op, u, v, z, 32, grid.dt, 3, sweeps=sweeps, coarse_tol=1e-2,
                           cycle_kind=kind)
    b = rng.standard_normal(h.levels[0].kkt.dim)
    xo = O.cycle(oh, 0, b)
    x1 = P.cycle(h, 0, b)
    assert rel(x1, xo) < 1e-10
    assert h.stats.iters == oh.coarse_iters
    assert rel(P.cycle(h, 0, b), xo) < 1e-10          # V: graph replay
    monkeypatch.setattr(M, "FUSED_PROLONG", False)
    h2 = P.build_hierarchy(p, u, v, z, grid, 3, sweeps=sweeps, coarse_tol=1e-2, cycle_kind=kind)
    assert rel(P.cycle(h2, 0, b), x1) < 1e-11


def test_dense_multi_sweep_fused_cycle_vs_oracle():
    import paper_2405_04808_b200 as P
    from oracle import tk_oracle as O
    from paper_2405_04808_b200 import multigrid as M
    n = 64
    grid = P.TimeGrid(5.0, n)
    vp = P.build_vanderpol(P.VanDerPolConfig(n_controls=1, u_init=(1.0, 0.0)), grid,
                           with_targets=False)
    rng = np.random.default_rng(5)
    zc = 0.3 * rng.standard_normal((n, 1))
    uv = P.forward_solve(vp, zc, grid).states
    h = P.build_hierarchy(vp, uv, uv, zc, grid, 4, sweeps=2)
    assert M.fused_vnn_ok(h, h.levels[0].kkt)
    oh = O.build_hierarchy(O.vanderpol(n_controls=1, u0=(1.0, 0.0)), uv, uv, zc, n, grid.dt, 4,
                           sweeps=2)
    b = rng.standard_normal(h.levels[0].kkt.dim)
    xo = O.cycle(oh, 0, b)
    assert rel(P.cycle(h, 0, b), xo) < 1e-10
    assert h.stats.iters == oh.coarse_iters
    assert rel(P.cycle(h, 0, b), xo) < 1e-10
