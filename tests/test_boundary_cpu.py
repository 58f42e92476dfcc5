"""CPU tests of the drop-in boundary's host logic (no device work):

* exception classes derive from the reference's when the package is imported
  from inside it (errors.py);
* the reference's StageBlocks field layout (kkt.py:53-80) from TRI diagonals;
* Theorem1Report semantics (kkt.py:496-517) and the SPD test (kkt.py:520-527);
* the BASELINE-shape golden fixtures are self-consistent (reference solves).
"""

import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, load_golden

REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "tempokkt")),
                    reason="reference not installed under baseline/_ref")
def test_exceptions_alias_reference_inside_drop_in():
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "import tempokkt\n"
        "import paper_2405_04808_b200 as P\n"
        "for n in ('SingularBlock','NonFiniteValue','Breakdown','DimensionMismatch',"
        "'IndivisibleSteps','NewtonDivergence','SingularMatrix','ConfigError'):\n"
        "    assert issubclass(getattr(P, n), getattr(tempokkt, n)), n\n"
        "try:\n"
        "    raise P.SingularBlock(7)\n"
        "except tempokkt.SingularBlock as e:\n"
        "    assert e.block_index == 7 and 'block 7' in str(e)\n"
        "print('ok')\n" % REF)
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    # standalone: plain classes, no reference import
    code2 = ("import sys, paper_2405_04808_b200 as P\n"
             "assert 'tempokkt' not in sys.modules\n"
             "assert P.SingularBlock.__mro__[2] is Exception\n")
    out = subprocess.run([sys.executable, "-c", code2], cwd=ROOT, capture_output=True, text=True)
    assert out.returncode == 0, out.stderr


def test_tri_dense_roundtrip():
    from paper_2405_04808_b200.kkt import _tri_dense, _tri_diags
    rng = np.random.default_rng(0)
    n = 9
    a = np.diag(rng.random(n)) + np.diag(rng.random(n - 1), 1) + np.diag(rng.random(n - 1), -1)
    d = np.stack([_tri_diags(a), _tri_diags(2 * a)])
    full = _tri_dense(d)
    assert np.array_equal(full[0], a) and np.array_equal(full[1], 2 * a)


def test_theorem1_report_and_spd():
    from paper_2405_04808_b200.kkt import Theorem1Report, _is_spd
    ok = np.ones(4, dtype=bool)
    k = ok.copy(); k[2] = False
    qz = ok.copy(); qz[3] = False
    r = Theorem1Report(q_u_ok=ok, q_v_ok=ok, q_z_ok=qz, k_ok=k)
    assert not r.passed
    assert r.failures() == [("q_z", 3), ("k", 2)]        # reference order: q_u, q_v, q_z, k
    assert Theorem1Report(ok, ok, ok, ok).passed
    assert _is_spd(np.eye(3)) and not _is_spd(-np.eye(3))
    assert not _is_spd(np.array([[1.0, 2.0], [0.0, 1.0]]))          # not symmetric
    assert not _is_spd(np.zeros((2, 2)))


@pytest.mark.parametrize("name", ("cfg2_shape", "cfg3_shape", "cfg4_shape"))
def test_shape_goldens_consistent(name):
    """The fixtures carry what the GPU tests compare against: the reference's
    MG-FGMRES history starts at ||b|| and ends at its reported residual."""
    if not os.path.exists(os.path.join(GOLDEN, f"{name}.npz")):
        pytest.skip(f"{name}.npz not generated")
    g = load_golden(name)
    hist = g["fgmres_hist"]
    assert hist.shape == (int(g["fgmres_iters"]) + 1,)
    assert abs(hist[0] - np.linalg.norm(g["b"])) <= 1e-12 * hist[0]
    assert int(g["fgmres_coarse_calls"]) == int(g["fgmres_iters"])   # one V-cycle per iteration
    n, lv = int(g["n"]), int(g["levels"])
    assert n % (1 << (lv - 1)) == 0 and n >> (lv - 1) >= 2
