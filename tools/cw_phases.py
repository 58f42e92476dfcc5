"""Phase cycles of the warp chain (needs a -DTK_PROF build of tk_tri_chainw.cu):
python tools/cw_phases.py  (TK_LIB_PATH=... selects the variant)"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2405_04808_b200 as P  # noqa: E402
from paper_2405_04808_b200 import _lib, configs, device as dev  # noqa: E402
from paper_2405_04808_b200.smoothers import forward_subst  # noqa: E402

s = configs.build_setup(2)
h = P.build_hierarchy(s.problem, s.u, s.v, s.z, s.grid, s.levels, sweeps=1)
a = h.levels[-1].kkt
a.ensure_subst()
r = dev.to_device(__import__("numpy").random.default_rng(0).standard_normal(a.dim))
lib = _lib.load()
out = (ctypes.c_longlong * 8)()
for _ in range(3):
    forward_subst(a, r)
torch.cuda.synchronize()
ctypes.CDLL(os.environ.get("TK_LIB_PATH")).tk_debug_cw_prof(out)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    forward_subst(a, r)
e1.record()
torch.cuda.synchronize()
ctypes.CDLL(os.environ.get("TK_LIB_PATH")).tk_debug_cw_prof(out)
v = list(out)
print("forward_subst us", e0.elapsed_time(e1) * 100)
n = max(v[0], 1)
print("steps", v[0], "cycles/step", v[1] / n, "wait", v[2] / n, "rhs+sweeps", v[3] / n, "interface", v[4] / n,
      "backsub+out", v[5] / n)
