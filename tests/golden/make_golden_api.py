"""Golden vectors for the kkt-module helpers around the hot path, by the REAL
reference (run in the build container, the only place /root/reference exists):

    python tests/golden/make_golden_api.py

Reference code exercised: kkt.py:392-425 (split_parts), 428-470
(clustered_permutation / from_clustered / to_clustered), 473-493
(assemble_rhs), 546-560 (dump_matrix_market) on a van der Pol instance
(n_u = 2, n_z = 2, N = 6) whose linearisation point is stored, so the tests
rebuild the same stage blocks without the reference.
"""
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import tempokkt as tk  # noqa: E402
from tempokkt import kkt as K  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    n = 6
    g = tk.TimeGrid(1.5, n)
    p = tk.build_vanderpol(tk.VanDerPolConfig(), g)
    rng = np.random.default_rng(11)
    z = 0.3 * rng.standard_normal((n, p.n_z))
    u = tk.forward_solve(p, z, g).states
    v = u + 0.05 * rng.standard_normal(u.shape)
    st = K.build_stage_blocks(p, g.dt, u, v, z)
    a = K.assemble_kkt(st)
    dim = a.layout.dim
    x = rng.standard_normal(dim)
    d, low, up = K.split_parts(a)
    b1, b1v, b3, b4 = (rng.standard_normal((n, p.n_u)) for _ in range(4))
    b2 = rng.standard_normal((n, p.n_z))
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "a.mtx")
        K.dump_matrix_market(a, path)
        lines = open(path).read().splitlines()
    ent = np.array([[float(t) for t in ln.split()] for ln in lines[3:]])
    np.savez_compressed(
        os.path.join(HERE, "api_helpers.npz"),
        t_final=1.5, n=n, u=u, v=v, z=z, x=x,
        d_x=d(x), low_x=low(x), up_x=up(x), a_x=a.apply(x),
        perm=K.clustered_permutation(p.n_u, p.n_z, n),
        from_clustered=K.from_clustered(x, p.n_u, p.n_z, n),
        to_clustered=K.to_clustered(x, p.n_u, p.n_z, n),
        b1=b1, b1v=b1v, b2=b2, b3=b3, b4=b4, rhs=K.assemble_rhs(st, b1, b1v, b2, b3, b4),
        mm_header=np.array(lines[:3]), mm_entries=ent)
    print("api_helpers.npz", dim, ent.shape)


if __name__ == "__main__":
    main()
