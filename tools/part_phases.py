"""Per-phase cycles of the partitioned row kernel (CTA 0, thread 0), from a
-DTK_PROF build loaded through TK_LIB_PATH.  usage: python tools/part_phases.py [config]"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2405_04808_b200 as P  # noqa: E402
from paper_2405_04808_b200 import _lib, configs, device as dev  # noqa: E402
from paper_2405_04808_b200.smoothers import jacobi_sweeps  # noqa: E402

s = configs.build_setup(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
h = P.build_hierarchy(s.problem, s.u, s.v, s.z, s.grid, s.levels, sweeps=1)
a = h.levels[0].kkt
b = dev.to_device(s.rhs())
x = jacobi_sweeps(a, b, None, 1, 1.0)
lib = _lib.load()
buf = (ctypes.c_longlong * 10)()
lib.tk_debug_part_prof(buf)
for _ in range(3):
    y = jacobi_sweeps(a, b, x, 1, 1.0)
torch.cuda.synchronize()
lib.tk_debug_part_prof(buf)
names = ["-", "phase1", "chunk sweeps", "xch1", "rows", "pcr", "E", "xch3", "output", "end barrier"]
tot = sum(buf[i] for i in range(1, 10))
rows = 3 * ((a.n_steps + 1 + 295) // 296)
for i in range(1, 10):
    print(f"{names[i]:14s} {buf[i] / rows:9.0f} cycles/row  {100 * buf[i] / tot:5.1f}%")
print("total cycles/row", tot / rows)
