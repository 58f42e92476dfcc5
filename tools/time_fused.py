"""Time the fused V(1,1) kernels of configs[N] (fine level): python tools/time_fused.py [cfg] [tag]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2405_04808_b200 as P
from paper_2405_04808_b200 import configs, device as dev, roofline
from paper_2405_04808_b200.multigrid import TransferOps
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
tag = sys.argv[2] if len(sys.argv) > 2 else "x"
s = configs.build_setup(cfg)
a = P.assemble_kkt(P.build_stage_blocks(s.problem, s.grid.dt, s.u, s.v, s.z))
t = TransferOps(a.n_steps, a.n_steps // 2, a.n_u, a.n_z)
b = dev.to_device(s.rhs())
x, rc, y = dev.empty(a.dim), dev.empty(t.coarse_dim), dev.empty(a.dim)
ec = dev.to_device(np.random.default_rng(1).standard_normal(t.coarse_dim))
def run(name, *args):
    for _ in range(3):
        dev.call(name, *args)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        dev.call(name, *args)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    byts = roofline.algorithmic_bytes(name, args)
    print(f"{tag} {name}: {ms:.4f} ms  {byts / ms / 1e6:.0f} GB/s  frac {byts / ms / 1e6 / 6547:.3f}")
run("tk_jacobi0_restrict_um", a.lref, dev.P(b), dev.P(x), dev.P(rc), dev.stream())
run("tk_jacobi_prolong", a.lref, dev.P(b), dev.P(x), dev.P(ec), dev.P(y), dev.stream())
run("tk_jacobi_sweep", a.lref, dev.P(b), dev.P(x), dev.P(y), 1.0, dev.stream())
