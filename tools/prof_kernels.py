"""One fine-level call of each HBM-bound hot kernel on configs[N] (default 2):
KKT apply (tri_apply<0>), Jacobi sweep with x (tri_rows_part), fused
residual-restrict (tri_resrestrict), prolong-add (prolong_rows_kernel) --
for `ncu --set full` captures.  Not a benchmark."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2405_04808_b200 as P  # noqa: E402
from paper_2405_04808_b200 import configs, device as dev  # noqa: E402
from paper_2405_04808_b200.smoothers import jacobi_sweeps  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
s = configs.build_setup(cfg)
h = P.build_hierarchy(s.problem, s.u, s.v, s.z, s.grid, 2, sweeps=1)
a = h.levels[0].kkt
t = h.transfers[0]
b = dev.to_device(s.rhs())
x0 = jacobi_sweeps(a, b, None, 1, 1.0)          # (warm-up: D^-1 b)
torch.cuda.synchronize()
y = a.apply(x0)                                   # tri_apply<0>
x1 = jacobi_sweeps(a, b, x0, 1, 1.0)              # tri_rows_part, x present
rc = dev.empty(t.coarse_dim)
work = dev.empty(a.dim)
dev.call("tk_residual_restrict", a.lref, dev.P(b), dev.P(x1), dev.P(rc), dev.P(work), dev.stream())
t.prolong_add(rc, x1)                             # prolong_rows_kernel
dev.call("tk_residual_restrict_jacobi0", a.lref, dev.P(b), dev.P(x0), 1.0, dev.P(rc),
         dev.stream())                            # restrict_jacobi0_rows (x0 = D^-1 b)
x2 = dev.empty(a.dim)
dev.call("tk_jacobi0_restrict", a.lref, dev.P(b), 1.0, dev.P(x2), dev.P(rc),
         dev.stream())                            # tri_rows_part<..., RJ>: sweep + restriction
from paper_2405_04808_b200 import _lib  # noqa: E402
if a.family == 1 and _lib.load().tk_jacobi_prolong_ok(a.lref, 1.0):
    x3 = dev.empty(a.dim)
    dev.call("tk_jacobi0_restrict_um", a.lref, dev.P(b), dev.P(x3), dev.P(rc),
             dev.stream())                        # ... storing only u / mu (V(1,1) pre-smoothing)
    ec = dev.to_device(__import__("numpy").random.default_rng(5).standard_normal(t.coarse_dim))
    x4 = dev.empty(a.dim)
    dev.call("tk_jacobi_prolong", a.lref, dev.P(b), dev.P(x3), dev.P(ec), dev.P(x4),
             dev.stream())                        # tri_rows_part<..., PR>: prolongation + post-smoothing
torch.cuda.synchronize()
print("ok", s.describe())
