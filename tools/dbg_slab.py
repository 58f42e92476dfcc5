"""Debug: single-GPU vs slab (2 virtual ranks) vs oracle FGMRES histories on the cfg1_burgers golden."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
import paper_2405_04808_b200 as P
from conftest import load_golden, product_problem, oracle_problem
from oracle import tk_oracle as O
from paper_2405_04808_b200 import slabs
g = load_golden("cfg1_burgers"); p, grid = product_problem(g)
u, v, z, b = g["u"], g["v"], g["z"], g["b"]
levels, R, its = 4, 2, 30
h = P.build_hierarchy(p, u, v, z, grid, levels, sweeps=int(g["sweeps"]), coarse_tol=1e-2)
from paper_2405_04808_b200 import krylov as KR
single_log = []
_arn = KR.DeviceSpace.arnoldi
def _arn_log(self, V, j, w):
    n_ = w.numel()
    if n_ == h.levels[0].kkt.dim:
        win = w.cpu().numpy().copy()
        hc = _arn(self, V, j, w)
        single_log.append((j, win, hc.copy(), V[j + 1].cpu().numpy().copy()))
        return hc
    return _arn(self, V, j, w)
KR.DeviceSpace.arnoldi = _arn_log
x1, rep1 = P.fgmres(h.levels[0].kkt.as_operator(), P.mg_preconditioner(h), b, rel_tol=1e-8, max_iters=its)
print("single coarse iters", h.stats.iters, h.stats.calls)
oh = O.build_hierarchy(oracle_problem(g), u, v, z, int(g["n"]), float(g["dt"]), levels, sweeps=int(g["sweeps"]), coarse_tol=1e-2)
xo, orep = O.fgmres(oh.levels[0].kkt.apply, O.mg_prec(oh), b, rel_tol=1e-8, max_iters=its)
print("oracle coarse iters", oh.coarse_iters, oh.coarse_calls)
d1 = np.abs(np.array(rep1.residual_history) / np.array(orep.history) - 1)
print("single vs oracle first bad idx", np.argmax(d1 > 1e-10) if (d1 > 1e-10).any() else None, d1.max())
comms = slabs.ThreadComm.group(R)
def body(c):
    sh = slabs.SlabHierarchy(p, u, v, z, grid, levels, c, sweeps=int(g["sweeps"]), coarse_tol=1e-2)
    off, ln = sh.local_span()
    bl = torch.from_numpy(np.ascontiguousarray(b[off:off + ln])).cuda()
    xs, rep = slabs.fgmres(sh, bl, rel_tol=1e-8, max_iters=its)
    torch.cuda.synchronize()
    st = sh.coarse.stats if sh.coarse is not None else None
    return off, xs.cpu().numpy(), rep, (st.iters, st.calls) if st else None
res = sorted(slabs.run_threads(comms, body), key=lambda t: t[0])
print("slab coarse iters", res[0][3])
d2 = np.abs(np.array(res[0][2].residual_history) / np.array(orep.history) - 1)
print("slab vs oracle first bad idx", np.argmax(d2 > 1e-10) if (d2 > 1e-10).any() else None, d2.max())

# ---- which operation diverges first?  record every slab V-cycle / operator application
print("--- per-call comparison against the single-GPU kernels")
comms = slabs.ThreadComm.group(R)
log = [dict(v=[], a=[]) for _ in range(R)]
def body2(c):
    sh = slabs.SlabHierarchy(p, u, v, z, grid, levels, c, sweeps=int(g["sweeps"]), coarse_tol=1e-2)
    off, ln = sh.local_span()
    vc, ap = sh.vcycle, sh.apply
    def vcycle(bl):
        out = vc(bl)
        log[c.rank]["v"].append((bl.cpu().numpy().copy(), out.cpu().numpy().copy()))
        return out
    def apply(xl):
        out = ap(xl)
        log[c.rank]["a"].append((xl.cpu().numpy().copy(), out.cpu().numpy().copy()))
        return out
    sh.vcycle, sh.apply = vcycle, apply
    mg = sh.be.mgs
    def mgs(comm, V, j, w):
        win = w.cpu().numpy().copy()
        Vin = V[:j + 1].cpu().numpy().copy()
        hc = mg(comm, V, j, w)
        log[c.rank].setdefault("m", []).append((Vin, win, hc.copy(), w.cpu().numpy().copy(), V[j + 1].cpu().numpy().copy()))
        return hc
    sh.be.mgs = mgs
    bl = torch.from_numpy(np.ascontiguousarray(b[off:off + ln])).cuda()
    xs, rep = slabs.fgmres(sh, bl, rel_tol=1e-8, max_iters=its)
    torch.cuda.synchronize()
    return off, rep
res = sorted(slabs.run_threads(comms, body2), key=lambda t: t[0])
a0 = h.levels[0].kkt
from paper_2405_04808_b200 import graph as G
G.ENABLED = False
nv = len(log[0]["v"])
for k in range(nv):
    vin = np.concatenate([log[r]["v"][k][0] for r in range(R)])
    vout = np.concatenate([log[r]["v"][k][1] for r in range(R)])
    ref = P.cycle(h, 0, vin)
    e = np.linalg.norm(vout - ref) / np.linalg.norm(ref)
    if e > 1e-12 or k < 2:
        print("vcycle call", k, "rel diff", e)
    if e > 1e-12:
        break
for k in range(len(log[0]["a"])):
    xin = np.concatenate([log[r]["a"][k][0] for r in range(R)])
    xout = np.concatenate([log[r]["a"][k][1] for r in range(R)])
    ref = a0.apply(xin)
    e = np.linalg.norm(xout - ref) / np.linalg.norm(ref)
    if e > 1e-13:
        print("apply call", k, "rel diff", e); break
for k in range(len(log[0]["m"])):
    Vin = np.concatenate([log[r]["m"][k][0] for r in range(R)], axis=1)
    win = np.concatenate([log[r]["m"][k][1] for r in range(R)])
    hc = log[0]["m"][k][2]
    w_ = win.copy(); href = np.zeros(len(hc))
    for i in range(Vin.shape[0]):
        href[i] = Vin[i] @ w_; w_ -= href[i] * Vin[i]
    href[-1] = np.linalg.norm(w_)
    e = np.abs(hc - href) / max(np.abs(href).max(), 1e-300)
    if e.max() > 1e-11:
        print("mgs call", k, "h mismatch", e, "h", hc, "ref", href)
        # per-rank partial dots of the first bad component
        i = int(np.argmax(e > 1e-11))
        for r in range(R):
            Vr, wr = log[r]["m"][k][0], log[r]["m"][k][1]
            print("  rank", r, "len", wr.size, "local <V_i,w> (w before any update)", Vr[i] @ wr)
        break
for k in range(min(len(log[0]["m"]), len(single_log))):
    win = np.concatenate([log[r]["m"][k][1] for r in range(R)])
    hc = log[0]["m"][k][2]
    vnext = np.concatenate([log[r]["m"][k][4] for r in range(R)])
    j_, win1, hc1, vnext1 = single_log[k]
    ew = np.linalg.norm(win - win1) / np.linalg.norm(win1)
    eh = np.abs(hc - hc1).max() / np.abs(hc1).max()
    ev = np.linalg.norm(vnext - vnext1) / np.linalg.norm(vnext1)
    if max(ew, eh, ev) > 1e-11:
        print("vs single: arnoldi call", k, "w_in diff", ew, "h diff", eh, "V[j+1] diff", ev)
        print("   h slab", hc, "h single", hc1)
        break
d3 = np.abs(np.array(res[0][1].residual_history) / np.array(orep.history) - 1)
print("second slab run vs oracle first bad idx", np.argmax(d3 > 1e-10) if (d3 > 1e-10).any() else None, d3.max())
