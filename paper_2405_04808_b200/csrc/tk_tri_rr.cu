// TRI family: fused residual + restriction, rc = R (b - A x)
// (multigrid.py:281-288 `restrict_kkt(b - a.apply(x))`, transfers
// multigrid.py:104-112).
//
// The restriction keeps the states/multipliers of the even fine time levels
// and averages the controls of each fine pair, so coarse block row c needs
// only the (v, mu, z) residual of fine row 2c and the (u, lam, z) residual
// of fine row 2c+1.  One CTA per coarse row computes exactly those
// components (the same arithmetic as tri_apply<T_RESIDUAL>) and writes the
// coarse row: the fine residual vector never goes through HBM and the half
// of it that the restriction discards is never computed.
#include "tk_tri.cuh"

namespace tk {

// fine residual components of node j (tri_apply<T_RESIDUAL> arithmetic)
struct FineRow {
    const double* Qv;
    const double* Qu;
    const double* K;
    const double* C;
    int64_t ov, ou, oz, om, ol;
    const double* uprev;
    const double* munext;
    bool has_vm, has_uzl;
    __device__ FineRow(const TView& V, const double* x, int i) {
        const Lay& L = V.lay;
        const int n = V.n;
        has_vm = i >= 1;
        has_uzl = i < L.N;
        Qv = (i == L.N) ? V.Ql : V.Qm;
        Qu = (i == L.N - 1) ? V.Ql : V.Qm;
        K = has_uzl ? V.Ki(i, n) : nullptr;
        C = (has_uzl && has_vm) ? V.Ci(i, n) : nullptr;
        const int64_t bs = V.sl.base;
        ov = L.off_v(i) - bs; ou = L.off_u(i) - bs; oz = L.off_z(i) - bs;
        om = L.off_mu(i) - bs; ol = L.off_l(i) - bs;
        uprev = V.sl.uprev(L, x, i);
        munext = V.sl.munext(L, x, i);
    }
};

__global__ void __launch_bounds__(256) tri_resrestrict(TView V, Lay Lc, int64_t cbase, int c0,
                                                       int c1, const double* __restrict__ b,
                                                       const double* __restrict__ x,
                                                       double* __restrict__ rc) {
    const Lay& L = V.lay;
    const int n = V.n;
    const double kap = V.kappa;
    const double* Qz = V.Qz;
    for (int c = c0 + blockIdx.x; c < c1; c += gridDim.x) {
        const int ie = 2 * c, io = 2 * c + 1;
        const FineRow E(V, x, ie);
        const bool odd = io < L.N;   // fine row 2c+1 exists with its (u, z, lam) part
        const FineRow O(V, x, odd ? io : ie);
        const int64_t cs = Lc.start(c) - cbase;
        const int64_t ccv = Lc.off_v(c) - Lc.start(c), ccu = Lc.off_u(c) - Lc.start(c),
                      ccz = Lc.off_z(c) - Lc.start(c), ccm = Lc.off_mu(c) - Lc.start(c),
                      ccl = Lc.off_l(c) - Lc.start(c);
        for (int j = threadIdx.x; j < n; j += blockDim.x) {
            double rze = 0.0, rzo = 0.0;
            if (E.has_vm) {   // v, mu of fine row 2c
                double av = tmv(E.Qv, n, x + E.ov, j) - x[E.om + j];
                if (E.C) av += tmtv(E.C, n, x + E.ol, j);
                double am = -x[E.ov + j];
                if (E.uprev) am += E.uprev[j];
                rc[cs + ccv + j] = b[E.ov + j] - av;
                rc[cs + ccm + j] = b[E.om + j] - am;
            }
            if (E.has_uzl) {  // z of fine row 2c
                const double az = tmv(Qz, n, x + E.oz, j) + kap * tmv(Qz, n, x + E.ol, j);
                rze = b[E.oz + j] - az;
            }
            if (odd) {        // u, z, lam of fine row 2c+1
                double au = tmv(O.Qu, n, x + O.ou, j) + tmtv(O.K, n, x + O.ol, j);
                if (O.munext) au += O.munext[j];
                const double az = tmv(Qz, n, x + O.oz, j) + kap * tmv(Qz, n, x + O.ol, j);
                double al = tmv(O.K, n, x + O.ou, j) + kap * tmv(Qz, n, x + O.oz, j);
                if (O.C) al += tmv(O.C, n, x + O.ov, j);
                rzo = b[O.oz + j] - az;
                rc[cs + ccu + j] = b[O.ou + j] - au;
                rc[cs + ccl + j] = b[O.ol + j] - al;
                rc[cs + ccz + j] = 0.5 * (rze + rzo);
            }
        }
    }
}

// fine slab [r0, r1) (r0 even; r1 even or N+1) -> coarse rows [r0/2, c1)
int tri_resrestrict_launch(const tk_level* Lv, const double* b, const double* x, double* rc,
                           cudaStream_t s) {
    TView V(Lv);
    const int N = Lv->n_steps;
    const int r0 = V.sl.r0, r1 = V.sl.r1;
    if ((N & 1) || (r0 & 1) || ((r1 & 1) && r1 != N + 1)) {
        set_error("tk_residual_restrict: N=%d and slab [%d, %d) must be even-aligned", N, r0, r1);
        return TK_ERR_ARG;
    }
    Lay Lc(N / 2, Lv->n_u, Lv->n_z);
    const int c0 = r0 / 2;
    const int c1 = (r1 == N + 1) ? N / 2 + 1 : r1 / 2;
    const int64_t cbase = Lc.start(c0);
    const int rows = c1 - c0;
    const int th = Lv->n_u >= 256 ? 256 : 128;
    tri_resrestrict<<<rows, th, 0, s>>>(V, Lc, cbase, c0, c1, b, x, rc);
    return check_launch("tri_resrestrict");
}

}  // namespace tk
