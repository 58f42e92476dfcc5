"""Kernel-wide span of ONE grouped-carry launch (needs a -DTK_PROF build via
TK_LIB_PATH): last CTA end - first CTA start, last CTA start - first start,
CTA 0's own duration (ns), for phases A and C of one forward substitution."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2405_04808_b200 as P
from paper_2405_04808_b200 import configs, device as dev, _lib
s = configs.build_setup(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
h = P.build_hierarchy(s.problem, s.u, s.v, s.z, s.grid, s.levels, sweeps=1)
a = h.levels[-1].kkt
r = dev.to_device(torch.randn(a.dim, dtype=torch.float64).numpy())
from paper_2405_04808_b200.smoothers import forward_subst
lib = _lib.load()
buf = (ctypes.c_longlong * 6)()
for _ in range(3):
    forward_subst(a, r); torch.cuda.synchronize()
    lib.tk_debug_span(buf)
    for m, name in ((0, "phase A"), (1, "phase C")):
        print(name, "(ns): span", buf[3 * m], "last start - first start", buf[3 * m + 1],
              "CTA 0", buf[3 * m + 2])
