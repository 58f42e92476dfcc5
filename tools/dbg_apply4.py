"""Debug: KKT apply time at configs[4] before / after the hierarchy exists."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2405_04808_b200 as P
from paper_2405_04808_b200 import configs, device as dev

def t_apply(a, x, y, tag):
    for _ in range(2):
        dev.call("tk_kkt_apply", a.lref, dev.P(x), dev.P(y), dev.stream())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        dev.call("tk_kkt_apply", a.lref, dev.P(x), dev.P(y), dev.stream())
    e1.record()
    torch.cuda.synchronize()
    print(tag, e0.elapsed_time(e1) / 5, "ms; allocated GB", torch.cuda.memory_allocated() / 2**30,
          "reserved", torch.cuda.memory_reserved() / 2**30, "ptrs", hex(x.data_ptr()), hex(y.data_ptr()), flush=True)

s = configs.build_setup(4)
S = s.solver
h = P.build_hierarchy(s.problem, s.u, s.v, s.z, s.grid, s.levels, sweeps=S["sweeps"], cycle_kind=S["cycle"], coarse_tol=S["coarse_tol"])
a = h.levels[0].kkt
r = dev.to_device(s.rhs())
y = dev.empty(a.dim)
t_apply(a, r, y, "after build_hierarchy")
prec = P.mg_preconditioner(h)
for _ in range(2):
    prec(r)
torch.cuda.synchronize()
t_apply(a, r, y, "after 2 V-cycles, old y")
y2 = dev.empty(a.dim)
t_apply(a, r, y2, "new y")
t_apply(a, y2, y, "x = previous y")
