"""HostPipeline: overlapped copy-in / V-cycle / copy-out gives, step by step,
exactly the results of the blocking path."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_pipeline_matches_serial():
    import torch

    import paper_2405_04808_b200 as P
    grid = P.TimeGrid(1.0, 32)
    p = P.build_burgers(P.BurgersConfig(n_elems=65, theta=1.0, u0_kind="sinstep"), grid)
    u = P.forward_solve(p, np.zeros((32, 64)), grid).states
    h = P.build_hierarchy(p, u, u, np.zeros((32, 64)), grid, 3, sweeps=1)
    prec = P.mg_preconditioner(h)
    dim = h.levels[0].kkt.dim
    rng = np.random.default_rng(5)
    rhs = [rng.standard_normal(dim) for _ in range(5)]
    prec(rhs[0])        # the first cycle runs eagerly, the rest replay the CUDA graph
    ref = [prec(r) for r in rhs]                      # numpy in -> numpy out
    ins = [torch.from_numpy(r).pin_memory() for r in rhs]
    outs = [torch.empty(dim, dtype=torch.float64).pin_memory() for _ in rhs]
    P.HostPipeline(prec, dim).run(ins, outs)
    torch.cuda.synchronize()
    for o, r in zip(outs, ref):
        assert np.array_equal(o.numpy(), r)
