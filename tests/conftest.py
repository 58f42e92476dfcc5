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
