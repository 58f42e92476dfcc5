"""GPU parity at the BASELINE.json configuration SHAPES against the REAL
reference (tests/golden/make_golden_shapes.py):

* cfg2_shape -- configs[2]'s n_u = 512, dt and 6-level hierarchy (nt = 64);
* cfg3_shape -- configs[3]'s van der Pol N_z = 1, dt and 10-level hierarchy
  (nt = 2^14), full MG-FGMRES to 1e-8;
* cfg4_shape -- configs[4]'s n_u = 2048 (2-CTA-cluster local solves, n_u = 2048
  Gauss-Seidel chain), dt, nu = 0.005 and random smooth control (nt = 4).

Same linearisation point as the reference (stored u, v, z), same rhs; the
operator, block-diagonal solve and Jacobi sweep to 1e-13/1e-11, one V-cycle
(eager and CUDA-graph replay) and the MG-FGMRES solve to 1e-10 with identical
outer and coarse iteration counts (multigrid.py:190-301, krylov.py:77-210).
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden, product_problem, rel

pytestmark = pytest.mark.gpu

SHAPES = ("cfg2_shape", "cfg3_shape", "cfg4_shape")


def _golden(name):
    if not os.path.exists(os.path.join(GOLDEN, f"{name}.npz")):
        pytest.skip(f"{name}.npz not generated")
    return load_golden(name)


def _hierarchy(g):
    import paper_2405_04808_b200 as P
    p, grid = product_problem(g)
    h = P.build_hierarchy(p, g["u"], g["v"], g["z"], grid, int(g["levels"]),
                          sweeps=int(g["sweeps"]), cycle_kind="v", coarse_tol=1e-2)
    return P, p, grid, h


@pytest.mark.parametrize("name", SHAPES)
def test_forward_march(name):
    """Our forward march (tk_forward_*_host) reproduces the reference's
    linearisation point at the shape's dt."""
    import paper_2405_04808_b200 as P
    g = _golden(name)
    p, grid = product_problem(g)
    u = P.forward_solve(p, g["z"], grid).states
    assert rel(u, g["u"]) < 1e-12


@pytest.mark.parametrize("name", ("cfg2_shape", "cfg4_shape"))
def test_fine_level_ops(name):
    P, p, grid, h = _hierarchy(_golden(name))
    g = load_golden(name)
    a = h.levels[0].kkt
    assert rel(a.apply(g["x"]), g["Ax"]) < 1e-13
    assert rel(h.levels[0].dsolve.solve_all(g["b"]), g["Dinv_b"]) < 1e-11
    assert rel(P.jacobi_apply(a, h.levels[0].dsolve, g["b"], g["x"], 1), g["jac1"]) < 1e-11


@pytest.mark.parametrize("name", SHAPES)
def test_vcycle(name):
    """One V-cycle from zero: the eager cycle and the graph replay."""
    g = _golden(name)
    P, p, grid, h = _hierarchy(g)
    for k in range(2):                      # 1st eager (warm), 2nd the CUDA graph
        h.stats = type(h.stats)()
        x = P.cycle(h, 0, g["b"])
        assert h.stats.iters == int(g["cycle_v_coarse_iters"]), k
        assert rel(x, g["cycle_v"]) < 1e-10, k


@pytest.mark.parametrize("name", SHAPES)
def test_mg_fgmres(name):
    g = _golden(name)
    P, p, grid, h = _hierarchy(g)
    h.stats = type(h.stats)()
    x, rep = P.fgmres(h.levels[0].kkt.as_operator(), P.mg_preconditioner(h), g["b"],
                      rel_tol=1e-8, max_iters=int(g["fgmres_max_iters"]))
    assert rep.iterations == int(g["fgmres_iters"])
    assert h.stats.calls == int(g["fgmres_coarse_calls"])
    assert h.stats.iters == int(g["fgmres_coarse_iters"])
    hist = np.array(rep.residual_history)
    assert hist.shape == g["fgmres_hist"].shape
    assert np.max(np.abs(hist - g["fgmres_hist"]) / g["fgmres_hist"][0]) < 1e-10
    assert rel(x, g["fgmres_x"]) < 1e-10
    assert abs(rep.final_relative_residual - float(g["fgmres_rel"])) <= 1e-10
