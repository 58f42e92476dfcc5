"""Probe the TRI row kernels at large n_u: which kernel runs, its time, and
the identity D (D^{-1} b) = b.  usage: python tools/large_n_probe.py 2048 [nt]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_04808_b200 as P  # noqa: E402
from paper_2405_04808_b200 import roofline  # noqa: E402

nu = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
nt = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
grid = P.TimeGrid(1.0, nt)
p = P.build_burgers(P.BurgersConfig(n_elems=nu + 1, theta=1.0, u0_kind="sinstep"), grid)
u = P.forward_solve(p, np.zeros((nt, nu)), grid).states
st = P.build_stage_blocks(p, grid.dt, u, u, np.zeros((nt, nu)))
a = P.assemble_kkt(st)
rng = np.random.default_rng(0)
b = torch.from_numpy(rng.standard_normal(a.dim)).cuda()
x = torch.from_numpy(rng.standard_normal(a.dim)).cuda()
y = P.jacobi_apply(a, None, b, x, 1)
r = a.residual(b, x)
e = (a.apply_diag(y - x) - r).norm() / r.norm()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    P.jacobi_apply(a, None, b, x, 1)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
byts = roofline.algorithmic_bytes("tk_jacobi_sweep", (a.lref, 0, 1, 0, 1.0))
print(f"n_u={nu} nt={nt}: identity err {float(e):.2e}  jacobi {ms:.3f} ms  {byts / ms / 1e6:.0f} GB/s")
