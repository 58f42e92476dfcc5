import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
CASES = ("vdp_ref", "vdp_cn", "burgers_ref", "cfg0_vdp", "cfg1_burgers")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run under gpurun)")
    config.addinivalue_line("markers", "slow: longer CPU test")


def load_golden(name):
    with np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False) as f:
        return {k: f[k] for k in f.files}


def oracle_problem(g):
    """Rebuild the oracle problem matching a golden case's parameters."""
    from oracle import tk_oracle as O
    if "n_controls" in g:
        return O.vanderpol(mu=float(g["mu"]), alpha=float(g["alpha"]),
                           n_controls=int(g["n_controls"]), u0=tuple(g["u0"]),
                           theta=float(g["theta"]))
    return O.burgers(n_u=int(g["n_u"]), nu=float(g["nu"]), alpha=float(g["alpha"]),
                     theta=float(g["theta"]), u0_kind=str(g["u0_kind"]))


@pytest.fixture(params=CASES)
def golden_case(request):
    return request.param, load_golden(request.param)


def product_problem(g):
    """The product-side ProblemSpec + TimeGrid for a golden case."""
    import paper_2405_04808_b200 as P
    n, T = int(g["n"]), float(g["t_final"])
    grid = P.TimeGrid(T, n)
    if "n_controls" in g:
        cfg = P.VanDerPolConfig(mu=float(g["mu"]), alpha=float(g["alpha"]),
                                u_init=tuple(g["u0"]), n_controls=int(g["n_controls"]))
        return P.build_vanderpol(cfg, grid, theta=float(g["theta"]), with_targets=False), grid
    cfg = P.BurgersConfig(nu=float(g["nu"]), alpha=float(g["alpha"]), n_elems=int(g["n_u"]) + 1,
                          theta=float(g["theta"]), u0_kind=str(g["u0_kind"]))
    return P.build_burgers(cfg, grid), grid


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def have_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
