"""Timeline of HostPipeline on configs[2]: per-step start/end of the copy-in,
the V-cycle and the copy-out (CUDA events on each stream)."""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import paper_2405_04808_b200 as P  # noqa: E402
from paper_2405_04808_b200 import configs, device as dev, pipeline  # noqa: E402

s = configs.build_setup(2)
S = s.solver
h = P.build_hierarchy(s.problem, s.u, s.v, s.z, s.grid, s.levels, sweeps=1, coarse_tol=1e-2)
prec = P.mg_preconditioner(h)
r = torch.from_numpy(s.rhs()).pin_memory()
outs = [torch.empty_like(r).pin_memory() for _ in range(2)]
ev = []
orig_prec = prec


def timed_prec(x):
    a = torch.cuda.Event(enable_timing=True); a.record()
    y = orig_prec(x)
    b = torch.cuda.Event(enable_timing=True); b.record()
    ev.append((a, b))
    return y


pipe = P.HostPipeline(timed_prec, s.dim)
n = 8
pipe.run([r] * 2, outs)
torch.cuda.synchronize()
ev.clear()
e0 = torch.cuda.Event(enable_timing=True); e0.record()
import time
t0 = time.perf_counter()
pipe.run([r] * n, [outs[k & 1] for k in range(n)])
host_ms = (time.perf_counter() - t0) * 1e3
e1 = torch.cuda.Event(enable_timing=True); e1.record()
torch.cuda.synchronize()
print(f"total {e0.elapsed_time(e1) / n:.2f} ms/step (host enqueue+sync {host_ms / n:.2f})")
for k, (a, b) in enumerate(ev):
    print(f"step {k}: V-cycle {e0.elapsed_time(a):8.2f} -> {e0.elapsed_time(b):8.2f}")
