"""Phase timestamps of one chain step (needs a -DTK_PROF build via TK_LIB_PATH)."""
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
from paper_2405_04808_b200.smoothers import forward_subst, backward_subst
for fn in (forward_subst, backward_subst):
    fn(a, r); torch.cuda.synchronize()
    lib = _lib.load(); lib.tk_debug_prof.restype = ctypes.c_int
    buf = (ctypes.c_longlong * 16)()
    lib.tk_debug_prof(buf)
    t = [buf[i] for i in range(7)]
    print(fn.__name__, "n", a.n_u, "phases(cycles):", [t[i + 1] - t[i] for i in range(6)], "total", t[6] - t[0])
