"""Debug: V-cycle time of two hierarchies built one after the other in one process."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2405_04808_b200 as P
from paper_2405_04808_b200 import configs, device as dev
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
keep = []
for rep in range(5):
    s = configs.build_setup(cfg)
    S = s.solver
    h = P.build_hierarchy(s.problem, s.u, s.v, s.z, s.grid, s.levels, sweeps=S["sweeps"], cycle_kind=S["cycle"], coarse_tol=S["coarse_tol"])
    r = dev.to_device(s.rhs())
    prec = P.mg_preconditioner(h)
    for k in range(3):
        prec(r)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(10):
        prec(r)
    e1.record()
    torch.cuda.synchronize()
    print(rep, "ms/cycle", e0.elapsed_time(e1) / 10, "mem", torch.cuda.memory_allocated() >> 20, "MB", flush=True)
    if os.environ.get("KEEP") == "1":
        keep.append((h, prec, r))
    del h, prec, r
    if os.environ.get('GC') == '1':
        import gc; gc.collect(); torch.cuda.synchronize(); torch.cuda.empty_cache()
