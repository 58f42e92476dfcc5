"""Pin the CPU oracle to golden vectors produced by the real reference
(tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from conftest import oracle_problem
from oracle import tk_oracle as O


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _setup(g):
    p = oracle_problem(g)
    n, dt = int(g["n"]), float(g["dt"])
    st = O.build_stages(p, dt, g["u"], g["v"], g["z"])
    a = O.Kkt(st)
    return p, n, dt, st, a, O.DiagSolve(a)


def test_forward_solve(golden_case):
    name, g = golden_case
    p = oracle_problem(g)
    n, dt = int(g["n"]), float(g["dt"])
    z = g["z"] if name.startswith("cfg") else np.zeros((n, p.n_z))
    states = O.forward_solve(p, z, n, dt)
    assert rel(states, g["fwd_states"]) < 1e-13


def test_stages_and_operator(golden_case):
    name, g = golden_case
    p, n, dt, st, a, d = _setup(g)
    for k, ref in (("k", "K"), ("c", "C"), ("b", "B"), ("q_u", "Qu"), ("q_v", "Qv"),
                   ("q_z", "Qz")):
        assert rel(getattr(st, k), g[ref]) < 1e-15, k
    assert rel(a.apply(g["x"]), g["Ax"]) < 1e-14
    assert rel(d.all(g["b"]), g["Dinv_b"]) < 1e-13
    # dense materialisation oracle of the apply (kkt.py:262-276)
    if a.dim <= 3000:
        assert rel(a.materialize() @ g["x"], g["Ax"]) < 1e-13


def test_smoothers(golden_case):
    name, g = golden_case
    p, n, dt, st, a, d = _setup(g)
    b, x = g["b"], g["x"]
    assert rel(O.jacobi(a, d, b, x, 1), g["jac1"]) < 1e-13
    assert rel(O.jacobi(a, d, b, x, 2), g["jac2"]) < 1e-13
    assert rel(O.fgs(a, d, b, x), g["fgs"]) < 1e-12
    assert rel(O.bgs(a, d, b, x), g["bgs"]) < 1e-12
    assert rel(O.sgs(a, d, b, x), g["sgs"]) < 1e-12
    assert rel(O.sgs(a, d, b, np.zeros_like(x)), g["sgs0"]) < 1e-12


def _hier(g, cycle_kind="v"):
    p = oracle_problem(g)
    return O.build_hierarchy(p, g["u"], g["v"], g["z"], int(g["n"]), float(g["dt"]),
                             int(g["levels"]), sweeps=int(g["sweeps"]),
                             cycle_kind=cycle_kind, coarse_tol=1e-2)


def test_transfers_and_coarse(golden_case):
    name, g = golden_case
    h = _hier(g)
    lf, lc = h.levels[0].kkt.lay, h.levels[1].kkt.lay
    assert np.array_equal(O.restrict_kkt(lf, lc, g["x"]), g["restrict_x"])
    assert np.array_equal(O.prolong_kkt(lf, lc, g["xc"]), g["prolong_xc"])
    # restrict o prolong = identity (multigrid.py:8-10)
    assert np.array_equal(O.restrict_kkt(lf, lc, O.prolong_kkt(lf, lc, g["xc"])), g["xc"])
    xcs = O.coarse_solve(h, g["coarse_r"])
    assert h.coarse_iters == int(g["coarse_iters"])
    assert rel(xcs, g["coarse_x"]) < 1e-11


@pytest.mark.parametrize("kind", ["v", "w", "f"])
def test_cycles(golden_case, kind):
    name, g = golden_case
    h = _hier(g, kind)
    out = O.cycle(h, 0, g["b"])
    assert h.coarse_iters == int(g[f"cycle_{kind}_coarse_iters"])
    assert rel(out, g[f"cycle_{kind}"]) < 1e-10


@pytest.mark.parametrize("outer", ["fgmres", "gmres"])
def test_full_solve(golden_case, outer):
    name, g = golden_case
    if name.startswith("cfg") and outer == "gmres":
        pytest.skip("401-iteration GMRES solve pinned through fgmres only (CPU time)")
    h = _hier(g)
    a = h.levels[0].kkt
    fn = O.fgmres if outer == "fgmres" else O.gmres
    x, rep = fn(a.apply, O.mg_prec(h), g["b"], rel_tol=1e-8, max_iters=401)
    assert rep.iterations == int(g[f"{outer}_iters"])
    assert h.coarse_calls == int(g[f"{outer}_coarse_calls"])
    assert h.coarse_iters == int(g[f"{outer}_coarse_iters"])
    hist = np.array(rep.history)
    assert hist.shape == g[f"{outer}_hist"].shape
    assert rel(hist, g[f"{outer}_hist"]) < 1e-8
    assert rel(x, g[f"{outer}_x"]) < 1e-8


def test_heat_neumann_oracle_vs_reference():
    """The oracle on the reference's heat-Neumann problem (general dense
    blocks, N_z = 1) against the reference-generated golden
    (tests/golden/make_golden_heat.py): operator, local solves, smoothers,
    transfers, one V-cycle and the FGMRES iteration count / history."""
    from conftest import load_golden
    g = load_golden("heat_ref")
    n, levels = int(g["n"]), int(g["levels"])
    p = O.heat_neumann(n_cells=int(g["n_cells"]))
    dt = 1.0 / n
    st = O.build_stages(p, dt, g["u"], g["v"], g["z"])
    assert rel(st.k[0], g["k0"]) < 1e-15 and rel(st.c[1], g["c1"]) < 1e-15
    assert rel(st.b[0], g["b0"]) < 1e-15 and rel(st.q_u[0], g["q_u0"]) < 1e-15
    a = O.Kkt(st)
    d = O.DiagSolve(a)
    x, b = g["x"], g["b"]
    assert rel(a.apply(x), g["apply"]) < 1e-14
    assert rel(d.all(b), g["solve_all"]) < 1e-12
    assert rel(O.jacobi(a, d, b, x, 2, 1.0), g["jacobi2"]) < 1e-12
    assert rel(O.jacobi(a, d, b, x, 1, 0.7), g["jacobi_w"]) < 1e-12
    assert rel(O.fgs(a, d, b, x), g["fgs"]) < 1e-12
    assert rel(O.sgs(a, d, b, x), g["sgs"]) < 1e-12
    h = O.build_hierarchy(p, g["u"], g["v"], g["z"], n, dt, levels, sweeps=1, coarse_tol=1e-2)
    assert rel(O.cycle(h, 0, b), g["cycle"]) < 1e-11
    xs, rep = O.fgmres(h.levels[0].kkt.apply, O.mg_prec(h), b, rel_tol=1e-8, max_iters=40)
    assert rep.iterations == int(g["fgmres_iters"])
    assert np.allclose(rep.history, g["fgmres_hist"], rtol=1e-10, atol=0)
    assert rel(xs, g["fgmres_x"]) < 1e-10
