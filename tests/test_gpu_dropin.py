"""GPU: the package-level drop-in of INTEGRATION.md §1 applied to the
reference's own SQP driver, and the reference's singularity exceptions.

* ``tempokkt.sqp.AugmentedSystem`` (sqp.py:186-213, 316-343) with its
  imports switched to this package runs ``sqp_solve`` (sqp.py:415-531) on a
  reference-built van der Pol ProblemSpec (no ``native`` tag: the generic
  stage path) and reproduces the unmodified reference run: every augmented
  solve has the same FGMRES iteration count and residual history (1e-10 of
  its initial residual), the same solution, and the SQP iterates agree.
* ``build_hierarchy(check=True)`` raises SingularBlock with the reference's
  stage index for a singular K_i (multigrid.py:221-226, kkt.py:530-543);
  ``check=False`` builds; a singular diagonal block raises SingularBlock
  with the reference's block index (kkt.py:347-368).

The reference package is the pip-installed copy under baseline/_ref (it
travels to the GPU box with the repo); the tests skip when it is absent.
"""

import os
import sys

import numpy as np
import pytest

from conftest import ROOT, rel

pytestmark = pytest.mark.gpu

SWAP = ("build_stage_blocks", "assemble_kkt", "build_hierarchy", "default_levels",
        "mg_preconditioner", "fgmres", "gmres")


def _reference():
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "tempokkt")):
        pytest.skip("reference package not installed under baseline/_ref")
    if path not in sys.path:
        sys.path.insert(0, path)
    import tempokkt
    return tempokkt


def _run_sqp(tk, p, g, swap: bool, iters: int):
    import tempokkt.sqp as S
    import paper_2405_04808_b200 as P
    saved = {nm: getattr(S, nm) for nm in SWAP}
    calls = []

    def recorder(fn):
        def run(*a, **kw):
            x, rep = fn(*a, **kw)
            calls.append((rep.iterations, np.array(rep.residual_history),
                          rep.final_relative_residual, np.array(x, copy=True)))
            return x, rep
        return run

    try:
        if swap:
            for nm in SWAP:
                setattr(S, nm, getattr(P, nm))
        S.fgmres, S.gmres = recorder(S.fgmres), recorder(S.gmres)
        res = tk.sqp_solve(p, g, tk.SqpConfig(max_sqp_iters=iters), tk.SolverConfig())
    finally:
        for nm, fn in saved.items():
            setattr(S, nm, fn)
    return res, calls


def test_reference_sqp_with_swapped_imports():
    tk = _reference()
    g = tk.TimeGrid(8.0, 64)
    p = tk.build_vanderpol(tk.VanDerPolConfig(), g)       # reference ProblemSpec
    assert not hasattr(p, "native")
    ref, ref_calls = _run_sqp(tk, p, g, swap=False, iters=3)
    our, our_calls = _run_sqp(tk, p, g, swap=True, iters=3)
    assert len(our_calls) == len(ref_calls) > 0
    for k, ((ri, rh, rr, rx), (oi, oh, orr, ox)) in enumerate(zip(ref_calls, our_calls)):
        assert oi == ri, (k, oi, ri)
        assert oh.shape == rh.shape
        assert np.max(np.abs(oh - rh)) <= 1e-10 * rh[0], k
        assert rel(ox, rx) < 1e-9, k
    assert our.iterations == ref.iterations
    assert our.ls_calls == ref.ls_calls and our.ls_iters == ref.ls_iters
    assert our.coarse_calls == ref.coarse_calls and our.coarse_iters == ref.coarse_iters
    for f in ("u", "v", "z", "lam", "mu"):
        assert rel(getattr(our.state, f), getattr(ref.state, f)) < 1e-9, f


def test_stage_blocks_host_views():
    """The reference's StageBlocks fields (kkt.py:53-80) on our StageBlocks,
    for a reference-built spec (generic path) and the native builders."""
    tk = _reference()
    import paper_2405_04808_b200 as P
    from tempokkt import kkt as RK
    g = tk.TimeGrid(1.0, 16)
    pr = tk.build_burgers(tk.BurgersConfig(n_elems=17, theta=1.0), g)
    u = tk.forward_solve(pr, np.zeros((16, 16)), g).states
    z = 0.1 * np.random.default_rng(0).standard_normal((16, 16))
    ref = RK.build_stage_blocks(pr, g.dt, u, u, z)
    ours = P.build_stage_blocks(pr, g.dt, u, u, z)                 # generic path
    gp = P.TimeGrid(1.0, 16)
    nat = P.build_burgers(P.BurgersConfig(n_elems=17, theta=1.0), gp)
    native = P.build_stage_blocks(nat, gp.dt, u, u, z)             # device linearisation
    for st in (ours, native):
        for f in ("k", "c", "b", "q_u", "q_v", "q_z"):
            assert getattr(st, f).shape == getattr(ref, f).shape, f
            assert np.array_equal(getattr(st, f), getattr(ref, f)), f


def _singular_vdp(P, n_controls=2, fz=None):
    """van der Pol with mu = 2.5, dt = 0.5: K_i = -I + dt F_u(u_i) is exactly
    singular where u_i[0] = 0 (det = 1 - dt mu + dt^2 = 0)."""
    mu = 2.5
    grid = P.TimeGrid(8.0, 16)
    u = np.random.default_rng(5).uniform(0.5, 1.5, (16, 2))
    u[5] = (0.0, 0.7)
    z = np.zeros((16, n_controls))
    fz = np.eye(2) if fz is None else fz
    spec = P.ProblemSpec(
        n_u=2, n_z=n_controls, mass=np.eye(2),
        f_eval=lambda uu, zz: np.array([uu[1], mu * (1 - uu[0] ** 2) * uu[1] - uu[0]]) + fz @ zz,
        f_jac_u=lambda uu, zz: np.array([[0.0, 1.0], [-2 * mu * uu[0] * uu[1] - 1.0,
                                                      mu * (1 - uu[0] ** 2)]]),
        f_jac_z=lambda uu, zz: fz, u0=np.array([1.0, 0.0]), theta=1.0, dt=grid.dt,
        u_target=np.zeros((16, 2)), z_target=np.zeros((16, n_controls)), w_state=np.eye(2),
        w_control=0.1 * np.eye(n_controls))
    return spec, grid, u, z


def test_singular_k_raises_singular_block():
    import paper_2405_04808_b200 as P
    spec, grid, u, z = _singular_vdp(P)
    with pytest.raises(P.SingularBlock) as exc:
        P.build_hierarchy(spec, u, u, z, grid, 2, check=True)
    assert exc.value.block_index == 5
    h = P.build_hierarchy(spec, u, u, z, grid, 2, check=False)  # B keeps the blocks regular
    assert h.n_levels == 2
    try:
        tk = _reference()
    except pytest.skip.Exception:
        return
    from tempokkt import multigrid as RM, timedisc as RT
    rspec = RT.ProblemSpec(**{f: getattr(spec, f) for f in (
        "n_u", "n_z", "mass", "f_eval", "f_jac_u", "f_jac_z", "u0", "theta", "dt",
        "u_target", "z_target", "w_state", "w_control")})
    with pytest.raises(tk.SingularBlock) as rexc:
        RM.build_hierarchy(rspec, u, u, z, tk.TimeGrid(8.0, 16), 2, check=True)
    assert rexc.value.block_index == exc.value.block_index
    RM.build_hierarchy(rspec, u, u, z, tk.TimeGrid(8.0, 16), 2, check=False)


def test_singular_diagonal_block():
    """F_z = (2, 1)^T spans the left null space's complement of the singular
    K_5, so [K_5 B_5] loses rank and diagonal block 5 is singular: the
    reference's DiagonalSolver raises SingularBlock(5) even with check=False."""
    import paper_2405_04808_b200 as P
    fz = np.array([[1.0], [0.5]])      # K_5 = [[-1, .5], [-.5, .25]]: y = (.5, -1), y.fz = 0
    spec, grid, u, z = _singular_vdp(P, n_controls=1, fz=fz)
    with pytest.raises(P.SingularBlock) as exc:
        P.build_hierarchy(spec, u, u, z, grid, 2, check=False)
    assert exc.value.block_index == 5
    try:
        tk = _reference()
    except pytest.skip.Exception:
        return
    from tempokkt import multigrid as RM, timedisc as RT
    rspec = RT.ProblemSpec(**{f: getattr(spec, f) for f in (
        "n_u", "n_z", "mass", "f_eval", "f_jac_u", "f_jac_z", "u0", "theta", "dt",
        "u_target", "z_target", "w_state", "w_control")})
    with pytest.raises(tk.SingularBlock) as rexc:
        RM.build_hierarchy(rspec, u, u, z, tk.TimeGrid(8.0, 16), 2, check=False)
    assert rexc.value.block_index == 5
