"""Time the fine-level KKT apply of configs[N] with CUDA events: python tools/time_apply.py [cfg]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2405_04808_b200 as P  # noqa: E402
from paper_2405_04808_b200 import configs, device as dev, roofline  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
s = configs.build_setup(cfg)
st = P.build_stage_blocks(s.problem, s.grid.dt, s.u, s.v, s.z)
a = P.assemble_kkt(st)
x = dev.to_device(s.rhs())
y = dev.empty(a.dim)
byts = roofline.algorithmic_bytes("tk_kkt_apply", (a.lref,))
for tag, xin in (("random", x), ("smooth", torch.linspace(0, 1, a.dim, dtype=torch.float64, device="cuda"))):
    for _ in range(3):
        dev.call("tk_kkt_apply", a.lref, dev.P(xin), dev.P(y), dev.stream())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    K = 10
    for _ in range(K):
        dev.call("tk_kkt_apply", a.lref, dev.P(xin), dev.P(y), dev.stream())
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    print(f"{tag}: {ms:.4f} ms/apply  {byts / ms / 1e6:.0f} GB/s  threads={os.environ.get('TK_APPLY_THREADS', 'default')}")
