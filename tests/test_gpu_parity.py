"""GPU parity: every hot-path operation of libtempokkt_b200.so against the
golden vectors of the real reference (tests/golden) and the CPU oracle.
Run on a B200 (``pytest -m gpu``)."""

import numpy as np
import pytest

from conftest import CASES, load_golden, oracle_problem, product_problem, rel

pytestmark = pytest.mark.gpu

# fp64 parity tolerances (north star: 1e-10 relative on solutions/residuals)
TOL_OP = 1e-13      # single operator applications
TOL_SOLVE = 1e-11   # local KKT solves / smoother sweeps (different elimination order)
TOL_MG = 1e-10      # cycles, coarse solves and outer Krylov solutions


@pytest.fixture(scope="module", params=CASES)
def case(request):
    import paper_2405_04808_b200 as P
    g = load_golden(request.param)
    p, grid = product_problem(g)
    st = P.build_stage_blocks(p, grid.dt, g["u"], g["v"], g["z"])
    a = P.assemble_kkt(st)
    return request.param, g, p, grid, st, a


def _dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _host(x):
    return x.detach().cpu().numpy()


def test_stage_linearisation_bitwise(case):
    name, g, p, grid, st, a = case
    from paper_2405_04808_b200.kkt import FAMILY_DENSE, _tri_diags
    if st.family == FAMILY_DENSE:
        assert np.array_equal(_host(st.K), g["K"])
        assert np.array_equal(_host(st.C), g["C"])
        assert np.array_equal(_host(st.B), g["B"])
    else:
        kd = np.stack([_tri_diags(k) for k in g["K"]])
        cd = np.stack([_tri_diags(c) for c in g["C"]])
        assert np.array_equal(_host(st.K), kd)
        assert np.array_equal(_host(st.C), cd)


def test_operator_apply(case):
    name, g, p, grid, st, a = case
    assert rel(_host(a.apply(_dev(g["x"]))), g["Ax"]) < TOL_OP
    # numpy in -> numpy out (drop-in boundary)
    assert rel(a.apply(g["x"]), g["Ax"]) < TOL_OP
    r = _host(a.residual(_dev(g["b"]), _dev(g["x"])))
    assert rel(r, g["b"] - g["Ax"]) < TOL_OP


def test_generic_upload_path(case):
    """Reference-layout StageBlocks arrays -> same device operator."""
    import paper_2405_04808_b200 as P
    name, g, p, grid, st, a = case
    st2 = P.stage_blocks_from_arrays(g["K"], g["C"], g["B"], g["Qu"], g["Qv"], g["Qz"])
    a2 = P.assemble_kkt(st2)
    assert st2.family == st.family
    assert rel(a2.apply(g["x"]), g["Ax"]) < TOL_OP
    assert rel(P.DiagonalSolver(a2).solve_all(g["b"]), g["Dinv_b"]) < TOL_SOLVE


def test_block_diagonal(case):
    from oracle import tk_oracle as O
    import paper_2405_04808_b200 as P
    name, g, p, grid, st, a = case
    d = P.DiagonalSolver(a)
    assert rel(d.solve_all(g["b"]), g["Dinv_b"]) < TOL_SOLVE
    ost = O.build_stages(oracle_problem(g), float(g["dt"]), g["u"], g["v"], g["z"])
    oa = O.Kkt(ost)
    assert rel(a.apply_diag(g["x"]), oa.apply_diag(g["x"])) < TOL_OP
    # D (D^{-1} b) = b
    y = d.solve_all(_dev(g["b"]))
    assert rel(_host(a.apply_diag(y)), g["b"]) < TOL_SOLVE


def test_smoothers(case):
    import paper_2405_04808_b200 as P
    name, g, p, grid, st, a = case
    b, x = g["b"], g["x"]
    assert rel(P.jacobi_apply(a, None, b, x, 1), g["jac1"]) < TOL_SOLVE
    assert rel(P.jacobi_apply(a, None, b, x, 2), g["jac2"]) < TOL_SOLVE
    assert rel(P.fgs_apply(a, None, b, x), g["fgs"]) < TOL_SOLVE
    assert rel(P.bgs_apply(a, None, b, x), g["bgs"]) < TOL_SOLVE
    assert rel(P.sgs_apply(a, None, b, x), g["sgs"]) < TOL_SOLVE
    assert rel(P.sgs_apply(a, None, b, np.zeros_like(x)), g["sgs0"]) < TOL_SOLVE
    # fixed point: b = A x  =>  one sweep returns x
    bx = a.apply(x)
    assert rel(P.jacobi_apply(a, None, bx, x, 1), x) < 1e-13


def _hier(g, p, grid, kind="v"):
    import paper_2405_04808_b200 as P
    return P.build_hierarchy(p, g["u"], g["v"], g["z"], grid, int(g["levels"]),
                             sweeps=int(g["sweeps"]), cycle_kind=kind, coarse_tol=1e-2)


def test_transfers_exact(case):
    name, g, p, grid, st, a = case
    h = _hier(g, p, grid)
    t = h.transfers[0]
    assert np.array_equal(t.restrict_kkt(g["x"]), g["restrict_x"])
    assert np.array_equal(t.prolong_kkt(g["xc"]), g["prolong_xc"])
    assert np.array_equal(t.restrict_kkt(t.prolong_kkt(g["xc"])), g["xc"])
    ones = np.ones(t.fine_dim)
    assert np.array_equal(t.restrict_kkt(ones), np.ones(t.coarse_dim))


def test_coarse_solve(case):
    import paper_2405_04808_b200 as P
    name, g, p, grid, st, a = case
    h = _hier(g, p, grid)
    x = P.coarse_solve(h, g["coarse_r"])
    assert h.stats.iters == int(g["coarse_iters"])
    assert rel(x, g["coarse_x"]) < TOL_MG


@pytest.mark.parametrize("kind", ["v", "w", "f"])
def test_cycles(case, kind):
    import paper_2405_04808_b200 as P
    name, g, p, grid, st, a = case
    h = _hier(g, p, grid, kind)
    out = P.cycle(h, 0, g["b"])
    assert h.stats.iters == int(g[f"cycle_{kind}_coarse_iters"])
    assert rel(out, g[f"cycle_{kind}"]) < TOL_MG


@pytest.mark.parametrize("outer", ["fgmres", "gmres"])
def test_full_solve(case, outer):
    import paper_2405_04808_b200 as P
    name, g, p, grid, st, a = case
    h = _hier(g, p, grid)
    fn = P.fgmres if outer == "fgmres" else P.gmres
    x, rep = fn(h.levels[0].kkt.as_operator(), P.mg_preconditioner(h), g["b"],
                rel_tol=1e-8, max_iters=401)
    assert rep.iterations == int(g[f"{outer}_iters"])
    assert h.stats.calls == int(g[f"{outer}_coarse_calls"])
    assert h.stats.iters == int(g[f"{outer}_coarse_iters"])
    hist = np.array(rep.residual_history)
    assert hist.shape == g[f"{outer}_hist"].shape
    assert rel(hist, g[f"{outer}_hist"]) < TOL_MG
    assert rel(x, g[f"{outer}_x"]) < TOL_MG
    assert abs(rep.final_relative_residual - float(g[f"{outer}_rel"])) <= \
        TOL_MG * max(1.0, float(g[f"{outer}_rel"]))
