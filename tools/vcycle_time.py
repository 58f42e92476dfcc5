"""V-cycle time of configs[N] (default 2) with the per-call split of the
coarse substitutions; for sweeping env knobs (TK_CARRY, TK_CHAIN_CHUNK, ...).
usage: python tools/vcycle_time.py [cfg] [tag]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_04808_b200 as P  # noqa: E402
from paper_2405_04808_b200 import configs, device as dev  # noqa: E402

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 2
tag = sys.argv[2] if len(sys.argv) > 2 else "x"
s = configs.build_setup(idx)
S = s.solver
h = P.build_hierarchy(s.problem, s.u, s.v, s.z, s.grid, s.levels, sweeps=S["sweeps"],
                      cycle_kind=S["cycle"], coarse_tol=S["coarse_tol"])
r = dev.to_device(s.rhs())
prec = P.mg_preconditioner(h)
for _ in range(3):
    out = prec(r)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
K = 20
e0.record()
for _ in range(K):
    out = prec(r)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / K
dev.INSTR.timed, dev.INSTR.records = {"tk_forward_subst", "tk_backward_subst", "tk_sgs_back_half"}, []
prec(r)
torch.cuda.synchronize()
per = {}
for nm, a, t0, t1 in dev.INSTR.records:
    per.setdefault(nm, []).append(t0.elapsed_time(t1))
dev.INSTR.timed = None
np.save(f"/tmp/vc_{tag}.npy", out.cpu().numpy()[::101])
print(f"{tag}: V-cycle {ms:.3f} ms  " + "  ".join(f"{k} {np.mean(v) * 1e3:.0f}us x{len(v)}"
                                                 for k, v in per.items()), flush=True)
