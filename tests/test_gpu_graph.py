"""The CUDA-graph V-cycle (graph.py, csrc/tk_graph.cu: levels 1..L-1 with
the coarse SGS-GMRES as a device-side WHILE loop) against the eager,
host-driven cycle and the CPU oracle: same result (1e-13), same coarse
iteration counts, fallback to the eager path when the device loop flags."""

import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu


def _burgers(nt=128, nu=64, levels=3, sweeps=1, coarse_max=401):
    import paper_2405_04808_b200 as P
    grid = P.TimeGrid(1.0, nt)
    p = P.build_burgers(P.BurgersConfig(n_elems=nu + 1, theta=1.0, u0_kind="sinstep"), grid)
    z = np.zeros((nt, nu))
    u = P.forward_solve(p, z, grid).states
    h = P.build_hierarchy(p, u, u, z, grid, levels, sweeps=sweeps, cycle_kind="v",
                          coarse_max_iters=coarse_max)
    return h, (p, u, z, grid)


def _vdp(nt=256, levels=4):
    import paper_2405_04808_b200 as P
    grid = P.TimeGrid(5.0, nt)
    vp = P.build_vanderpol(P.VanDerPolConfig(n_controls=1, u_init=(1.0, 0.0)), grid,
                           with_targets=False)
    zc = (0.5 * np.sin(2 * np.pi * grid.dt * np.arange(1, nt + 1) / 5.0)).reshape(nt, 1)
    uv = P.forward_solve(vp, zc, grid).states
    return P.build_hierarchy(vp, uv, uv, zc, grid, levels, sweeps=1)


def _eager(h, b):
    from paper_2405_04808_b200 import graph as G
    on = G.ENABLED
    G.ENABLED = False
    try:
        import paper_2405_04808_b200 as P
        c0, i0 = h.stats.calls, h.stats.iters
        x = P.cycle(h, 0, b)
        return x, h.stats.calls - c0, h.stats.iters - i0
    finally:
        G.ENABLED = on


def _graphed(h, b):
    import paper_2405_04808_b200 as P
    c0, i0 = h.stats.calls, h.stats.iters
    x = P.cycle(h, 0, b)
    return x, h.stats.calls - c0, h.stats.iters - i0


@pytest.mark.parametrize("builder", ["burgers", "burgers_sweeps2", "burgers_L2", "vdp"])
def test_graph_cycle_equals_eager(builder):
    from paper_2405_04808_b200 import graph as G
    if builder == "burgers":
        h, _ = _burgers()
    elif builder == "burgers_sweeps2":
        h, _ = _burgers(sweeps=2)
    elif builder == "burgers_L2":
        h, _ = _burgers(levels=2)
    else:
        h = _vdp()
    rng = np.random.default_rng(7)
    for trial in range(3):
        b = rng.standard_normal(h.levels[0].kkt.dim)
        xe, ce, ie = _eager(h, b)
        h._graph_warm = True
        xg, cg, ig = _graphed(h, b)
        assert getattr(h, "_graph", None) is not None, "graph path did not run"
        assert cg == ce == 1 and ig == ie, (ce, ie, cg, ig)
        assert rel(xg, xe) < 1e-13
    assert isinstance(h._graph, G.VCycleGraph)


def test_graph_cycle_vs_oracle():
    import paper_2405_04808_b200 as P
    from oracle import tk_oracle as O
    h, (p, u, z, grid) = _burgers(nt=128, nu=64, levels=3)
    op = O.burgers(n_u=64, nu=1e-2, alpha=0.1, theta=1.0, u0_kind="sinstep")
    oh = O.build_hierarchy(op, u, u, z, 128, grid.dt, 3, sweeps=1, cycle_kind="v")
    h._graph_warm = True
    b = np.random.default_rng(3).standard_normal(h.levels[0].kkt.dim)
    x = P.cycle(h, 0, b)
    assert h._graph is not None
    xo = O.cycle(oh, 0, b)
    assert rel(x, xo) < 1e-10
    assert h.stats.iters == oh.coarse_iters


def test_graph_fallback_on_basis_overflow():
    """cap = 1 coarse column: the device loop flags, the cycle re-runs eagerly
    (its coarse solve through the coarse-only graph) with the same result and
    iteration count."""
    import paper_2405_04808_b200 as P
    from paper_2405_04808_b200 import graph as G
    h, _ = _burgers()
    b = np.random.default_rng(11).standard_normal(h.levels[0].kkt.dim)
    xe, ce, ie = _eager(h, b)
    assert ie > 1
    h._graph_warm = True
    h._graph = G.VCycleGraph(h, cap=1)
    xg, cg, ig = _graphed(h, b)
    assert cg == ce and ig == ie
    assert rel(xg, xe) < 1e-13
    assert getattr(h, "_cgraph", None) is not None


def test_coarse_graph_matches_host_gmres():
    """graphed_coarse (coarse-only graph, used for the level gathered on rank 0
    of the time-slab path) against the host-driven coarse GMRES."""
    import paper_2405_04808_b200 as P
    from paper_2405_04808_b200 import graph as G
    from paper_2405_04808_b200.multigrid import coarse_solve
    h, _ = _burgers(nt=64, levels=2)
    rng = np.random.default_rng(2)
    r = rng.standard_normal(h.levels[-1].kkt.dim)
    G.ENABLED = False
    try:
        xe = coarse_solve(h, r)
    finally:
        G.ENABLED = True
    ie = h.stats.iters
    xg = coarse_solve(h, r)            # eager (warm-up) -> sets _coarse_warm
    xg = coarse_solve(h, r)            # graph
    assert h._cgraph is not None
    assert h.stats.iters == 3 * ie and h.stats.calls == 3
    assert rel(xg, xe) < 1e-13


def test_graph_fgmres_solve_matches_eager():
    import paper_2405_04808_b200 as P
    from paper_2405_04808_b200 import graph as G
    h = _vdp(nt=256, levels=4)
    op = h.levels[0].kkt.as_operator()
    b = np.random.default_rng(5).standard_normal(h.levels[0].kkt.dim)
    G.ENABLED = False
    try:
        xe, re_ = P.fgmres(op, P.mg_preconditioner(h), b, rel_tol=1e-8, max_iters=60)
    finally:
        G.ENABLED = True
    ie = h.stats.iters
    h.stats.calls = h.stats.iters = 0
    xg, rg = P.fgmres(op, P.mg_preconditioner(h), b, rel_tol=1e-8, max_iters=60)
    assert h._graph is not None
    assert rg.iterations == re_.iterations
    assert h.stats.iters == ie
    assert rel(xg, xe) < 1e-10
    np.testing.assert_allclose(rg.residual_history, re_.residual_history, rtol=1e-8)
