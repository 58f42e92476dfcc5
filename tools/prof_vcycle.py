"""Short V-cycle driver for ncu captures: builds configs[N] (default 2) and
applies the V-cycle preconditioner a few times.  Not a benchmark."""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2405_04808_b200 as P  # noqa: E402
from paper_2405_04808_b200 import configs, device as dev  # noqa: E402


def main():
    idx = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    s = configs.build_setup(idx)
    S = s.solver
    h = P.build_hierarchy(s.problem, s.u, s.v, s.z, s.grid, s.levels, sweeps=S["sweeps"],
                          cycle_kind=S["cycle"], coarse_tol=S["coarse_tol"])
    r = dev.to_device(s.rhs())
    prec = P.mg_preconditioner(h)
    if os.environ.get("PROF_GRAPH") == "1":
        # eager warm-up cycle + graph capture, then ONE graphed cycle inside
        # cudaProfilerStart/Stop (ncu --profile-from-start off)
        for _ in range(2):
            prec(r)
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        for _ in range(reps):
            prec(r)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    else:
        for _ in range(reps):
            prec(r)
        torch.cuda.synchronize()
    print("ok", s.describe(), h.stats.calls, h.stats.iters)


if __name__ == "__main__":
    main()
