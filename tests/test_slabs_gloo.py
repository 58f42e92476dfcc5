"""Multi-process (world_size 2, gloo, CPU) test of the time-slab driver:
halo exchanges, coarse gather/scatter and distributed dots of
paper_2405_04808_b200.slabs, with a CPU test backend built from the oracle's
dense operator rows.  The distributed V-cycle must equal the oracle's
single-process V-cycle."""

import os
import socket

import numpy as np
import pytest
import torch

from conftest import load_golden, oracle_problem

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class OracleSlab:
    """A slab level on the CPU: rows [row0, row1) of an oracle Kkt."""

    def __init__(self, kkt, dsolve, rows):
        from paper_2405_04808_b200 import slabs
        self.k, self.d = kkt, dsolve
        self.n_steps, self.n_u, self.n_z = kkt.n, kkt.nu, kkt.nz
        self.row0, self.row1 = rows
        self.off, self.dim = slabs.slab_span(self.n_steps, self.n_u, self.n_z, *rows)
        self.halo_u = torch.zeros(self.n_u, dtype=torch.float64) if self.row0 > 0 else None
        self.halo_mu = torch.zeros(self.n_u, dtype=torch.float64) \
            if self.row1 <= self.n_steps else None

    def embed(self, x):
        """Global vector with the local slice and the halos at their offsets."""
        lay = self.k.lay
        g = np.zeros(lay.dim)
        g[self.off:self.off + self.dim] = x.numpy()
        if self.halo_u is not None:
            g[lay.rows["u"][self.row0 - 1]] = self.halo_u.numpy()   # u_{row0} in row0-1
        if self.halo_mu is not None:
            g[lay.rows["mu"][self.row1 - 1]] = self.halo_mu.numpy()  # mu_{row1} in row1
        return g


class OracleBackend:
    def __init__(self, prob):
        self.prob = prob

    def slab_level(self, p, dt, u, v, z, rows):
        from oracle import tk_oracle as O
        st = O.build_stages(self.prob, dt, u, v, z)
        a = O.Kkt(st)
        return OracleSlab(a, O.DiagSolve(a), rows)

    def full_coarse(self, p, dt, u, v, z, coarse_tol, coarse_max_iters):
        from oracle import tk_oracle as O
        n = u.shape[0]
        return O.build_hierarchy(self.prob, u, v, z, n, dt, 1, coarse_tol=coarse_tol,
                                 coarse_max_iters=coarse_max_iters)

    def to_local(self, x):
        return torch.as_tensor(np.asarray(x, dtype=np.float64))

    def empty(self, n):
        return torch.zeros(n, dtype=torch.float64)

    def zeros(self, n):
        return torch.zeros(n, dtype=torch.float64)

    def halos(self, a):
        return a.halo_u, a.halo_mu

    def _rows_of(self, a, y):
        return y[a.off:a.off + a.dim]

    def apply(self, a, x):
        return torch.from_numpy(self._rows_of(a, a.k.apply(a.embed(x))).copy())

    def jacobi(self, a, b, x, omega):
        bl = b.numpy()
        r = bl.copy() if x is None else bl - self._rows_of(a, a.k.apply(a.embed(x)))
        g = np.zeros(a.k.lay.dim)
        g[a.off:a.off + a.dim] = r
        dg = a.d.all(g)
        d = self._rows_of(a, dg)
        out = omega * d if x is None else x.numpy() + omega * d
        return torch.from_numpy(out.copy())

    def residual_restrict(self, a, b, x, coarse_len, jacobi0_omega=None):
        # the oracle backend always forms the full residual (the coupling-only
        # form after a zero-start sweep is the same vector in exact arithmetic)
        from oracle import tk_oracle as O
        r = b.numpy() - self._rows_of(a, a.k.apply(a.embed(x)))
        g = np.zeros(a.k.lay.dim)
        g[a.off:a.off + a.dim] = r
        lc = O.Layout(a.n_steps // 2, a.n_u, a.n_z)
        rc = O.restrict_kkt(a.k.lay, lc, g)
        from paper_2405_04808_b200 import slabs
        c0 = a.row0 // 2
        c1 = a.n_steps // 2 + 1 if a.row1 == a.n_steps + 1 else a.row1 // 2
        co, cl = slabs.slab_span(a.n_steps // 2, a.n_u, a.n_z, c0, c1)
        assert cl == coarse_len
        return torch.from_numpy(rc[co:co + cl].copy())

    def prolong_add(self, a, ec, hprev, hnext, x):
        from oracle import tk_oracle as O
        from paper_2405_04808_b200 import slabs
        nc, nu, nz = a.n_steps // 2, a.n_u, a.n_z
        lc = O.Layout(nc, nu, nz)
        c0 = a.row0 // 2
        c1 = nc + 1 if a.row1 == a.n_steps + 1 else a.row1 // 2
        co, cl = slabs.slab_span(nc, nu, nz, c0, c1)
        g = np.zeros(lc.dim)
        g[co:co + cl] = ec.numpy()
        if c0 > 0:   # previous slab's last coarse row: u_{c0}, lam_{c0}
            g[lc.rows["u"][c0 - 1]] = hprev.numpy()[:nu]
            g[lc.rows["lam"][c0 - 1]] = hprev.numpy()[nu:]
        if c1 <= nc:  # next slab's first coarse row: v_{c1}, mu_{c1}
            g[lc.rows["v"][c1 - 1]] = hnext.numpy()[:nu]
            g[lc.rows["mu"][c1 - 1]] = hnext.numpy()[nu:]
        pf = O.prolong_kkt(a.k.lay, lc, g)
        x += torch.from_numpy(pf[a.off:a.off + a.dim].copy())

    def coarse_solve(self, h, r):
        from oracle import tk_oracle as O
        return torch.from_numpy(O.coarse_solve(h, r.numpy()))

    def local_dot(self, x, y):
        return torch.tensor([float(np.dot(x.numpy(), y.numpy()))], dtype=torch.float64)

    # Krylov vector operations on slab vectors (slabs.SlabSpace) -- host torch
    # here; the CUDA backend runs the libtempokkt_b200.so kernels
    def scale_into(self, a, x, y):
        torch.mul(x, a, out=y)

    def axpy(self, a, x, y):
        y.add_(x, alpha=a)

    def rsub(self, b, y):
        torch.sub(b, y, out=y)

    def gemv_t_add(self, V, c, x):
        c = torch.as_tensor(np.asarray(c, dtype=np.float64))
        x.add_(V[:c.numel()].T @ c)

    def sq_norms(self, vecs):
        return torch.tensor([float(np.dot(v.numpy(), v.numpy())) for v in vecs],
                            dtype=torch.float64)

    def mgs(self, comm, V, j, w):
        h = torch.zeros(j + 2, dtype=torch.float64)
        for i in range(j + 1):
            h[i] = float(np.dot(V[i].numpy(), w.numpy()))
            comm.allreduce_sum(h[i:i + 1])
            w.sub_(V[i], alpha=float(h[i]))
        h[j + 1] = float(np.dot(w.numpy(), w.numpy()))
        comm.allreduce_sum(h[j + 1:j + 2])
        h[j + 1] = np.sqrt(float(h[j + 1]))
        if float(h[j + 1]) != 0.0:
            torch.div(w, float(h[j + 1]), out=V[j + 1])
        return h.numpy().copy()

    def finish(self):
        pass


def _worker(rank, world, port, name, levels, out):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist
    from conftest import load_golden as lg, oracle_problem as op, product_problem as pp
    from paper_2405_04808_b200 import slabs
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    g = lg(name)
    prob = op(g)
    p, grid = pp(g)
    sh = slabs.SlabHierarchy(p, g["u"], g["v"], g["z"], grid, levels, slabs.TorchComm(),
                             sweeps=int(g["sweeps"]), coarse_tol=1e-2,
                             backend=OracleBackend(prob))
    off, ln = sh.local_span()
    b = torch.from_numpy(np.ascontiguousarray(g["b"][off:off + ln]))
    x = torch.from_numpy(np.ascontiguousarray(g["x"][off:off + ln]))
    e = sh.vcycle(b)
    ax = sh.apply(x)
    d = sh.dot(x, b)
    # the sharded outer solve (row 13): FGMRES around the slab V-cycle
    xs, rep = slabs.fgmres(sh, b, rel_tol=1e-8, max_iters=40)
    # plain GMRES without a preconditioner, restarted, from a nonzero guess
    xg, repg = slabs.gmres(sh, None, b, x0=x, rel_tol=1e-3, max_iters=12, restart=5)
    np.savez(os.path.join(out, f"r{rank}.npz"), off=off, e=e.numpy(), ax=ax.numpy(), d=d,
             xs=np.asarray(xs), its=rep.iterations, hist=np.asarray(rep.residual_history),
             rel=rep.final_relative_residual, xg=np.asarray(xg), gits=repg.iterations,
             ghist=np.asarray(repg.residual_history))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("name,levels", [("cfg1_burgers", 4), ("vdp_ref", 3)])
def test_gloo_two_ranks_match_oracle(tmp_path, name, levels):
    import torch.multiprocessing as mp

    from oracle import tk_oracle as O
    g = load_golden(name)
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), name, levels, str(tmp_path)), nprocs=world,
             join=True)
    parts = sorted((dict(np.load(tmp_path / f"r{r}.npz")) for r in range(world)),
                   key=lambda d: int(d["off"]))
    e = np.concatenate([q["e"] for q in parts])
    ax = np.concatenate([q["ax"] for q in parts])
    prob = oracle_problem(g)
    h = O.build_hierarchy(prob, g["u"], g["v"], g["z"], int(g["n"]), float(g["dt"]), levels,
                          sweeps=int(g["sweeps"]), coarse_tol=1e-2)
    ref = O.cycle(h, 0, g["b"])
    assert np.abs(e - ref).max() <= 1e-12 * np.abs(ref).max()
    assert np.abs(ax - h.levels[0].kkt.apply(g["x"])).max() <= 1e-13 * np.abs(ax).max()
    assert abs(float(parts[0]["d"]) - float(np.dot(g["x"], g["b"]))) < 1e-9
    # sharded FGMRES == the oracle's single-process FGMRES: identical iteration
    # counts on every rank, residual history and solution within 1e-10
    xo, orep = O.fgmres(h.levels[0].kkt.apply, O.mg_prec(h), g["b"], rel_tol=1e-8, max_iters=40)
    xs = np.concatenate([q["xs"] for q in parts])
    for q in parts:
        assert int(q["its"]) == orep.iterations
        assert np.allclose(q["hist"], orep.history, rtol=1e-10, atol=0)
        assert np.array_equal(q["hist"], parts[0]["hist"])
    assert np.linalg.norm(xs - xo) <= 1e-10 * np.linalg.norm(xo)
    xgo, grep_ = O.gmres(h.levels[0].kkt.apply, None, g["b"], x0=g["x"], rel_tol=1e-3,
                         max_iters=12, restart=5)
    xg = np.concatenate([q["xg"] for q in parts])
    assert int(parts[0]["gits"]) == int(parts[1]["gits"]) == grep_.iterations
    assert np.allclose(parts[0]["ghist"], grep_.history, rtol=1e-10, atol=0)
    assert np.linalg.norm(xg - xgo) <= 1e-10 * np.linalg.norm(xgo)
