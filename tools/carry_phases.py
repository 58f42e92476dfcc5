"""Cycle buckets of the chunk carry (needs a -DTK_PROF build via TK_LIB_PATH):
[8] wait for U_{t-1}, [9] wait for the row block, [10] matvec + push,
[11] (grid variant) U load; grouped carry (tri_chain_carry_seg, phases A + C of
CTA 0): [12] wait for U_t, [13] wait for the row block, [14] matvec + push, [0] prologue, [1] store of the starts, [2] CTA barrier + next
TMA issue, [3] epilogue.
Accumulated over the steps of CTA 0."""
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
forward_subst(a, r); torch.cuda.synchronize()
lib = _lib.load(); lib.tk_debug_prof.restype = ctypes.c_int
buf = (ctypes.c_longlong * 16)()
lib.tk_debug_prof(buf)
b0 = [buf[i] for i in range(0, 16)]
forward_subst(a, r); torch.cuda.synchronize()
lib.tk_debug_prof(buf)
b1 = [buf[i] for i in range(0, 16)]
print("carry chunk", a.level.chain_chunk, "buckets(cycles, one launch):", [y - x for x, y in zip(b0, b1)])
