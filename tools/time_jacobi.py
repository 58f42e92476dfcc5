"""Time the fine-level Jacobi sweep of configs[N] (default 2) with CUDA events;
prints ms/sweep and the achieved algorithmic GB/s.  Saves the sweep output to
/tmp/jac_<tag>.npy for cross-variant comparison.  usage: python tools/time_jacobi.py [cfg] [tag]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_04808_b200 as P  # noqa: E402
from paper_2405_04808_b200 import configs, device as dev, roofline  # noqa: E402
from paper_2405_04808_b200.smoothers import jacobi_sweeps  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
tag = sys.argv[2] if len(sys.argv) > 2 else "x"
s = configs.build_setup(cfg)
st = P.build_stage_blocks(s.problem, s.grid.dt, s.u, s.v, s.z)
a = P.assemble_kkt(st)
b = dev.to_device(s.rhs())
x = jacobi_sweeps(a, b, None, 1, 1.0)
y = jacobi_sweeps(a, b, x, 1, 1.0)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(3):
    jacobi_sweeps(a, b, x, 1, 1.0, out=y)
e0.record()
K = 20
for _ in range(K):
    jacobi_sweeps(a, b, x, 1, 1.0, out=y)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / K
byts = roofline.algorithmic_bytes("tk_jacobi_sweep", (a.lref, 0, 1, 0, 1.0))
print(f"{tag}: {ms:.4f} ms/sweep  {byts / ms / 1e6:.0f} GB/s")
np.save(f"/tmp/jac_{tag}.npy", y.cpu().numpy()[:: 997])
