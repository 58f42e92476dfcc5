"""GPU: the fused Arnoldi step (tk_arnoldi_mgs) against the unfused
dot/axpy/nrm2/scale_into sequence of the same kernels, and MG-(F)GMRES with
it against the reference's golden solves (krylov.py:77-210)."""

import numpy as np
import pytest

from conftest import load_golden, product_problem, rel

pytestmark = pytest.mark.gpu


def _mk(n, k, seed):
    import torch
    g = torch.Generator().manual_seed(seed)
    V = torch.randn(k + 2, n, generator=g, dtype=torch.float64).cuda()
    w = torch.randn(n, generator=g, dtype=torch.float64).cuda()
    return V, w


@pytest.mark.parametrize("n", [1, 37, 151552, 151553, 1 << 20, 3_000_017])
@pytest.mark.parametrize("j", [0, 1, 5])
def test_arnoldi_step_bitwise(n, j):
    import torch
    from paper_2405_04808_b200.krylov import vec_ops
    ops = vec_ops()
    V, w = _mk(n, j, 1000 * j + n % 997)
    V2, w2 = V.clone(), w.clone()
    h = ops.arnoldi(V, j, w)
    ref = []
    for i in range(j + 1):
        hij = ops.dot(V2[i], w2)
        ref.append(hij)
        ops.axpy(-hij, V2[i], w2)
    hj1 = ops.nrm2(w2)
    ref.append(hj1)
    ops.scale_into(1.0 / hj1, w2, V2[j + 1])
    torch.cuda.synchronize()
    assert np.array_equal(h, np.array(ref))
    assert torch.equal(w, w2)
    assert torch.equal(V[j + 1], V2[j + 1])


@pytest.mark.parametrize("outer", ["fgmres", "gmres"])
def test_fused_solve_bitwise_and_golden(outer):
    """Whole MG-preconditioned solve with and without the fused step: same
    bits; and against the reference's golden solve of BASELINE configs[1]
    (reduced nx): identical iteration counts, 1e-10 solutions."""
    import paper_2405_04808_b200 as P
    from paper_2405_04808_b200 import krylov
    g = load_golden("cfg1_burgers")
    p, grid = product_problem(g)
    res = {}
    for fused in (True, False):
        krylov.FUSED_ARNOLDI = fused
        try:
            h = P.build_hierarchy(p, g["u"], g["v"], g["z"], grid, int(g["levels"]),
                                  sweeps=int(g["sweeps"]), cycle_kind="v", coarse_tol=1e-2)
            fn = P.fgmres if outer == "fgmres" else P.gmres
            x, rep = fn(h.levels[0].kkt.as_operator(), P.mg_preconditioner(h), g["b"],
                        rel_tol=1e-8, max_iters=401)
            res[fused] = (x, rep, h.stats.iters)
        finally:
            krylov.FUSED_ARNOLDI = True
    (x1, r1, c1), (x0, r0, c0) = res[True], res[False]
    assert np.array_equal(x1, x0)
    assert r1.iterations == r0.iterations and c1 == c0
    assert r1.iterations == int(g[f"{outer}_iters"])
    assert c1 == int(g[f"{outer}_coarse_iters"])
    assert rel(x1, g[f"{outer}_x"]) < 1e-10


def test_cfg1_full_size_solve_vs_reference():
    """BASELINE configs[1] at FULL size (Burgers nx=128, nt=1024, 4-level
    V(1,1), FGMRES 1e-8 / 401 its) against the record of the reference's own
    solve (tests/golden/make_cfg1_full.py, 29 min on the CPU): same outer and
    coarse iteration counts, residual history and solution fingerprint within
    1e-10."""
    import paper_2405_04808_b200 as P
    from paper_2405_04808_b200 import configs
    g = load_golden("cfg1_full_solve")
    s = configs.build_setup(1)
    S = s.solver
    h = P.build_hierarchy(s.problem, s.u, s.v, s.z, s.grid, s.levels, sweeps=S["sweeps"],
                          cycle_kind=S["cycle"], coarse_tol=S["coarse_tol"])
    b = s.rhs()
    assert abs(np.linalg.norm(b) - float(g["b_norm"])) <= 1e-12 * float(g["b_norm"])
    x, rep = P.fgmres(h.levels[0].kkt.as_operator(), P.mg_preconditioner(h), b,
                      rel_tol=S["rel_tol"], max_iters=S["max_iters"])
    assert rep.iterations == int(g["fgmres_iters"])
    assert h.stats.calls == int(g["coarse_calls"]) and h.stats.iters == int(g["coarse_iters"])
    hist = np.array(rep.residual_history)
    assert rel(hist, g["fgmres_hist"]) < 1e-10
    assert abs(rep.final_relative_residual - float(g["fgmres_rel"])) < 1e-10
    assert rel(x[::int(g["x_stride"])], g["x_sample"]) < 1e-10
    assert abs(np.linalg.norm(x) - float(g["x_norm"])) < 1e-10 * float(g["x_norm"])


@pytest.mark.parametrize("cfg,nt,nx", [(1, 256, 128), (0, 512, None)])
def test_jacobi0_residual_restrict(cfg, nt, nx):
    """The coupling-only residual-restrict after the zero-start pre-smoothing
    sweep (tk_residual_restrict_jacobi0) against the general fused
    residual-restrict: the V-cycles agree to roundoff, the coarse-solve
    iteration counts are identical (TRI and DENSE families)."""
    import paper_2405_04808_b200 as P
    from paper_2405_04808_b200 import configs, multigrid
    s = configs.build_setup(cfg, nt=nt, nx=nx, levels=3)
    b = s.rhs()
    out = {}
    for flag in (True, False):
        multigrid.JACOBI0_RESIDUAL = flag
        try:
            h = P.build_hierarchy(s.problem, s.u, s.v, s.z, s.grid, s.levels, sweeps=1,
                                  coarse_tol=1e-2)
            out[flag] = (P.cycle(h, 0, b), h.stats.iters)
        finally:
            multigrid.JACOBI0_RESIDUAL = True
    assert out[True][1] == out[False][1]
    assert rel(out[True][0], out[False][0]) < 1e-12
