"""Time-slab sharding on one GPU: R virtual ranks (threads) drive the slab
kernels with halo exchanges; the distributed V-cycle, operator and dots must
reproduce the single-slab path (row-local kernels => bitwise for the cycle)."""

import numpy as np
import pytest

from conftest import load_golden, product_problem

pytestmark = pytest.mark.gpu


def _setup(name):
    g = load_golden(name)
    p, grid = product_problem(g)
    return g, p, grid


@pytest.mark.parametrize("name,R,levels", [("cfg1_burgers", 2, 4), ("cfg1_burgers", 4, 4),
                                           ("cfg0_vdp", 2, 3), ("cfg0_vdp", 4, 3),
                                           ("burgers_ref", 2, 3)])
def test_virtual_ranks_match_single(name, R, levels):
    import torch

    import paper_2405_04808_b200 as P
    from paper_2405_04808_b200 import slabs
    g, p, grid = _setup(name)
    u, v, z, b = g["u"], g["v"], g["z"], g["b"]
    h = P.build_hierarchy(p, u, v, z, grid, levels, sweeps=int(g["sweeps"]), coarse_tol=1e-2)
    ref = P.cycle(h, 0, b)
    ref_ax = P.assemble_kkt(P.build_stage_blocks(p, grid.dt, u, v, z)).apply(g["x"])

    comms = slabs.ThreadComm.group(R)

    def body(c):
        sh = slabs.SlabHierarchy(p, u, v, z, grid, levels, c, sweeps=int(g["sweeps"]),
                                 coarse_tol=1e-2)
        off, ln = sh.local_span()
        bl = torch.from_numpy(np.ascontiguousarray(b[off:off + ln])).cuda()
        xl = torch.from_numpy(np.ascontiguousarray(g["x"][off:off + ln])).cuda()
        out = sh.vcycle(bl)
        ax = sh.apply(xl)
        d = sh.dot(xl, bl)
        torch.cuda.synchronize()
        return off, out.cpu().numpy(), ax.cpu().numpy(), d

    res = slabs.run_threads(comms, body)
    got = np.concatenate([r[1] for r in sorted(res, key=lambda t: t[0])])
    ax = np.concatenate([r[2] for r in sorted(res, key=lambda t: t[0])])
    assert got.shape == ref.shape
    # (several sweeps: both cycles form the restricted residual from the couplings
    # of the last update, tk_jacobi_restrict -- the slabs with the two-phase
    # boundary fix-up tk_restrict_fix_slab_x)
    assert np.array_equal(got, ref), np.abs(got - ref).max()
    assert np.array_equal(ax, ref_ax)
    d = res[0][3]
    assert abs(d - float(np.dot(g["x"], b))) <= 1e-12 * abs(np.dot(np.abs(g["x"]), np.abs(b)))


@pytest.mark.parametrize("name,R,levels", [("cfg1_burgers", 2, 4), ("cfg0_vdp", 4, 3)])
def test_sharded_fgmres_matches_single_and_oracle(name, R, levels):
    """The outer MG-FGMRES over time slabs (slabs.fgmres: distributed MGS with
    device-resident allreduced dots) against the single-GPU solve and the
    oracle: identical iteration counts, history and solution within 1e-10."""
    import torch

    import paper_2405_04808_b200 as P
    from conftest import oracle_problem
    from oracle import tk_oracle as O
    from paper_2405_04808_b200 import slabs
    g, p, grid = _setup(name)
    u, v, z, b = g["u"], g["v"], g["z"], g["b"]
    its = 30
    h = P.build_hierarchy(p, u, v, z, grid, levels, sweeps=int(g["sweeps"]), coarse_tol=1e-2)
    x1, rep1 = P.fgmres(h.levels[0].kkt.as_operator(), P.mg_preconditioner(h), b,
                        rel_tol=1e-8, max_iters=its)
    oh = O.build_hierarchy(oracle_problem(g), u, v, z, int(g["n"]), float(g["dt"]), levels,
                           sweeps=int(g["sweeps"]), coarse_tol=1e-2)
    xo, orep = O.fgmres(oh.levels[0].kkt.apply, O.mg_prec(oh), b, rel_tol=1e-8, max_iters=its)
    comms = slabs.ThreadComm.group(R)

    def body(c):
        sh = slabs.SlabHierarchy(p, u, v, z, grid, levels, c, sweeps=int(g["sweeps"]),
                                 coarse_tol=1e-2)
        off, ln = sh.local_span()
        bl = torch.from_numpy(np.ascontiguousarray(b[off:off + ln])).cuda()
        xs, rep = slabs.fgmres(sh, bl, rel_tol=1e-8, max_iters=its)
        torch.cuda.synchronize()
        return off, xs.cpu().numpy(), rep

    res = sorted(slabs.run_threads(comms, body), key=lambda t: t[0])
    xs = np.concatenate([r[1] for r in res])
    for _, _, rep in res:
        assert rep.iterations == rep1.iterations == orep.iterations
        assert rep.residual_history == res[0][2].residual_history
        assert np.allclose(rep.residual_history, orep.history, rtol=1e-10, atol=0)
    assert np.linalg.norm(xs - x1) <= 1e-10 * np.linalg.norm(x1)
    assert np.linalg.norm(xs - xo) <= 1e-10 * np.linalg.norm(xo)


def test_slab_transfers_and_halo_checks():
    import torch

    from paper_2405_04808_b200 import _lib, slabs
    from paper_2405_04808_b200 import device as dev
    lib = _lib.load()
    N, nu, nz = 16, 2, 1
    m = 4 * nu + nz
    rng = np.random.default_rng(0)
    xf = rng.standard_normal(N * m)
    xc = rng.standard_normal((N // 2) * m)
    # whole-level restrict / prolong
    full_r = dev.empty((N // 2) * m)
    dev.call("tk_restrict", N, nu, nz, dev.P(dev.to_device(xf)), dev.P(full_r), dev.stream())
    full_p = dev.to_device(xf).clone()
    dev.call("tk_prolong_add", N, nu, nz, dev.P(dev.to_device(xc)), dev.P(full_p), dev.stream())
    for r0, r1 in ((0, 8), (8, 17), (4, 12)):
        fo, fl = slabs.slab_span(N, nu, nz, r0, r1)
        c0, c1 = r0 // 2, (N // 2 + 1) if r1 == N + 1 else r1 // 2
        co, cl = slabs.slab_span(N // 2, nu, nz, c0, c1)
        rc = dev.empty(cl)
        dev.call("tk_restrict_slab", N, nu, nz, r0, r1, dev.P(dev.to_device(xf[fo:fo + fl])),
                 dev.P(rc), dev.stream())
        assert np.array_equal(dev.to_host(rc), dev.to_host(full_r)[co:co + cl])
        # prolong with halos taken from the global coarse vector
        hp = np.zeros(2 * nu)
        hn = np.zeros(2 * nu)
        if r0 > 0:
            o_u = slabs.row_start(N // 2, nu, nz, c0 - 1) + (0 if c0 - 1 == 0 else nu)
            o_l = slabs.row_start(N // 2, nu, nz, c0 - 1) + (nu + nz if c0 - 1 == 0
                                                              else 3 * nu + nz)
            hp = np.concatenate([xc[o_u:o_u + nu], xc[o_l:o_l + nu]])
        if r1 <= N:
            base = slabs.row_start(N // 2, nu, nz, c1)
            o_v = base
            o_m = base + (nu if c1 == N // 2 else 2 * nu + nz)
            hn = np.concatenate([xc[o_v:o_v + nu], xc[o_m:o_m + nu]])
        xl = dev.to_device(xf[fo:fo + fl]).clone()
        xcl, hpd, hnd = (dev.to_device(a) for a in (xc[co:co + cl], hp, hn))  # keep alive
        dev.call("tk_prolong_add_slab", N, nu, nz, r0, r1, dev.P(xcl), dev.P(hpd), dev.P(hnd),
                 dev.P(xl), dev.stream())
        assert np.array_equal(dev.to_host(xl), dev.to_host(full_p)[fo:fo + fl])
    # odd slab edges are rejected
    bad = dev.empty(8)
    assert lib.tk_restrict_slab(N, nu, nz, 1, 8, dev.P(bad), dev.P(bad), None) == _lib.TK_ERR_ARG
    torch.cuda.synchronize()


@pytest.mark.parametrize("n_u,R,sweeps", [(512, 2, 1), (512, 4, 1), (100, 2, 1), (2048, 2, 1),
                                         (512, 2, 2), (100, 4, 3)])
def test_fused_pair_on_slabs_bitwise(n_u, R, sweeps):
    """The slab cycle runs V(1,1) through the fused pair (tk_jacobi0_restrict_um
    + tk_restrict_fix_slab after the halo exchange, tk_jacobi_prolong_slab with
    the coarse halos; reference multigrid.py:285-299 on a time slab): bitwise
    equal to the single-GPU fused cycle, which is pinned to the oracle.  sweeps > 1:
    tk_jacobi_restrict + the two-phase boundary fix-up tk_restrict_fix_slab_x."""
    import torch

    import paper_2405_04808_b200 as P
    from paper_2405_04808_b200 import slabs
    nt, levels = 32, 3
    grid = P.TimeGrid(1.0, nt)
    p = P.build_burgers(P.BurgersConfig(n_elems=n_u + 1, theta=0.5, u0_kind="sinstep"), grid)
    rng = np.random.default_rng(7)
    u = P.forward_solve(p, np.zeros((nt, n_u)), grid).states
    v = u + 0.01 * rng.standard_normal(u.shape)
    z = 0.1 * rng.standard_normal((nt, n_u))
    h = P.build_hierarchy(p, u, v, z, grid, levels, sweeps=sweeps, coarse_tol=1e-2)
    b = rng.standard_normal(h.levels[0].kkt.dim)
    ref = P.cycle(h, 0, b)
    comms = slabs.ThreadComm.group(R)
    used = []

    def body(c):
        sh = slabs.SlabHierarchy(p, u, v, z, grid, levels, c, sweeps=sweeps, coarse_tol=1e-2)
        used.append(all(sh.be.fused_pair_ok(a) for a in sh.levels))
        off, ln = sh.local_span()
        bl = torch.from_numpy(np.ascontiguousarray(b[off:off + ln])).cuda()
        out = sh.vcycle(bl)
        torch.cuda.synchronize()
        return off, out.cpu().numpy()

    res = slabs.run_threads(comms, body)
    assert all(used) and len(used) == R
    got = np.concatenate([r[1] for r in sorted(res, key=lambda t: t[0])])
    assert np.array_equal(got, ref), np.abs(got - ref).max()


@pytest.mark.parametrize("n_controls,R", [(1, 2), (2, 4)])
def test_dense_fused_pair_on_slabs_bitwise(n_controls, R):
    """van der Pol (DENSE family): the slab cycle through dense_rows_split with
    the coarse halos, bitwise against the single-GPU fused cycle."""
    import torch

    import paper_2405_04808_b200 as P
    from paper_2405_04808_b200 import slabs
    n, levels = 64, 3
    grid = P.TimeGrid(5.0, n)
    vp = P.build_vanderpol(P.VanDerPolConfig(n_controls=n_controls, u_init=(1.0, 0.0)), grid,
                           with_targets=False)
    rng = np.random.default_rng(11)
    zc = 0.3 * rng.standard_normal((n, n_controls))
    uv = P.forward_solve(vp, zc, grid).states
    vv = uv + 0.01 * rng.standard_normal(uv.shape)
    h = P.build_hierarchy(vp, uv, vv, zc, grid, levels, sweeps=1)
    b = rng.standard_normal(h.levels[0].kkt.dim)
    ref = P.cycle(h, 0, b)
    comms = slabs.ThreadComm.group(R)
    used = []

    def body(c):
        sh = slabs.SlabHierarchy(vp, uv, vv, zc, grid, levels, c, sweeps=1)
        used.append(all(sh.be.fused_pair_ok(a) for a in sh.levels))
        off, ln = sh.local_span()
        bl = torch.from_numpy(np.ascontiguousarray(b[off:off + ln])).cuda()
        out = sh.vcycle(bl)
        torch.cuda.synchronize()
        return off, out.cpu().numpy()

    res = slabs.run_threads(comms, body)
    assert all(used) and len(used) == R
    got = np.concatenate([r[1] for r in sorted(res, key=lambda t: t[0])])
    assert np.array_equal(got, ref), np.abs(got - ref).max()


def test_slab_pair_error_paths():
    """A slab level asks for its coarse halos (tk_jacobi_prolong -> TK_ERR_ARG
    without them); tk_restrict_fix_slab is a no-op on a whole level."""
    import torch

    import paper_2405_04808_b200 as P
    from paper_2405_04808_b200 import _lib, device as dev, slabs
    nt, n_u = 16, 128
    grid = P.TimeGrid(1.0, nt)
    p = P.build_burgers(P.BurgersConfig(n_elems=n_u + 1, theta=0.5, u0_kind="sinstep"), grid)
    u = P.forward_solve(p, np.zeros((nt, n_u)), grid).states
    z = np.zeros((nt, n_u))
    comms = slabs.ThreadComm.group(2)

    def body(c):
        sh = slabs.SlabHierarchy(p, u, u, z, grid, 2, c, sweeps=1)
        a = sh.levels[0]
        b = torch.randn(a.dim, dtype=torch.float64, device="cuda")
        x, y = dev.empty(a.dim), dev.empty(a.dim)
        ec = dev.zeros(sh.coarse_sizes[c.rank])
        rc = _lib.load().tk_jacobi_prolong(a.lref, dev.P(b), dev.P(x), dev.P(ec), dev.P(y),
                                           dev.stream())
        return rc

    assert all(rc == _lib.TK_ERR_ARG for rc in slabs.run_threads(comms, body))
    h = P.build_hierarchy(p, u, u, z, grid, 2, sweeps=1)
    a = h.levels[0].kkt
    rc = torch.full((h.transfers[0].coarse_dim,), 3.0, dtype=torch.float64, device="cuda")
    dev.call("tk_restrict_fix_slab", a.lref, dev.P(rc), dev.stream())
    torch.cuda.synchronize()
    assert bool((rc == 3.0).all())
