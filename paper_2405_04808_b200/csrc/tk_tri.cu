// TRI family: per-interval KKT blocks whose sub-blocks are tridiagonal in
// space (P1 finite elements, 1D Burgers: problems.py:425-473).
//
// One CTA owns one block row (time interval) of the Figure-3 operator.  The
// local KKT block (kkt.py:298-312) is solved exactly, without the dense
// (4nu+nz)^2 inverse of DiagonalSolver (kkt.py:338-389):
//   v   = -r_mu                                  (mu-row)
//   w   = Qz^{-1} r_z                            (scalar cyclic reduction, Qz constant)
//   [Qu  K^T     ] [u  ]   [r_u                        ]
//   [K  -k^2 Qz  ] [lam] = [r_lam - C v - k r_z        ]   (2x2-block cyclic reduction)
//   z   = w - k lam,   mu = Qv v + C^T lam - r_v
// using B = k Qz (k = kappa; Burgers: F_z = M, w_control = alpha M, k = 1/alpha).
// The (u,lam) system is symmetric quasi-definite, so cyclic reduction needs
// no pivoting.  All reductions run in shared memory (16 doubles per node).
#include "tk_common.cuh"

namespace tk {

struct TView {
    Lay lay;
    int n;
    const double* K;
    const double* C;
    const double* Qm;
    const double* Ql;
    const double* Qz;
    const double* cr;
    double kappa;
    TView(const tk_level* L)
        : lay(L->n_steps, L->n_u, L->n_z), n(L->n_u), K(L->K), C(L->C), Qm(L->Qm), Ql(L->Ql),
          Qz(L->Qz), cr(L->qz_cr), kappa(L->kappa) {}
};

// (A x)_j for a tridiagonal A stored [3][n] = (sub, diag, sup)
__device__ __forceinline__ double tmv(const double* A, int n, const double* x, int j) {
    double s = A[n + j] * x[j];
    if (j > 0) s += A[j] * x[j - 1];
    if (j < n - 1) s += A[2 * n + j] * x[j + 1];
    return s;
}
// (A^T x)_j
__device__ __forceinline__ double tmtv(const double* A, int n, const double* x, int j) {
    double s = A[n + j] * x[j];
    if (j > 0) s += A[2 * n + j - 1] * x[j - 1];
    if (j < n - 1) s += A[j + 1] * x[j + 1];
    return s;
}

static constexpr int kTriArrays = 16;

struct TriSm {
    double *Da, *Db, *Dc, *E0, *E1, *E2, *E3, *L0, *L1, *L2, *L3, *f0, *f1, *fw, *sv, *srv;
    __device__ TriSm(double* sm, int n) {
        double* p = sm;
        Da = p; p += n; Db = p; p += n; Dc = p; p += n;
        E0 = p; p += n; E1 = p; p += n; E2 = p; p += n; E3 = p; p += n;
        L0 = p; p += n; L1 = p; p += n; L2 = p; p += n; L3 = p; p += n;
        f0 = p; p += n; f1 = p; p += n; fw = p; p += n; sv = p; p += n; srv = p;
    }
};

// Block cyclic reduction of the symmetric quasi-definite 2x2-block tridiagonal
// system held in S (D sym (a,b,c), E upper coupling, f rhs), jointly with the
// scalar reduction of Qz w = fw using precomputed coefficients cr = [3][n]
// (inv_d, e_up, e_lo per node at its elimination level).  Solution overwrites f.
__device__ void cr_solve(int n, TriSm& S, const double* __restrict__ cr) {
    const int tid = threadIdx.x, nth = blockDim.x;
    const double* cinv = cr;
    const double* cup = cr + n;
    const double* clo = cr + 2 * n;
    const int top = 31 - __clz(n);
    for (int lev = 0; lev < top; ++lev) {
        const int s = 1 << lev;
        for (int m = tid;; m += nth) {
            const int p = s - 1 + 2 * s * m;
            if (p >= n) break;
            const double a = S.Da[p], b = S.Db[p], c = S.Dc[p];
            const double idet = 1.0 / (a * c - b * b);
            S.Da[p] = c * idet;
            S.Db[p] = -b * idet;
            S.Dc[p] = a * idet;
            if (p - s >= 0) {
                S.L0[p] = S.E0[p - s]; S.L1[p] = S.E1[p - s];
                S.L2[p] = S.E2[p - s]; S.L3[p] = S.E3[p - s];
            } else {
                S.L0[p] = 0.0; S.L1[p] = 0.0; S.L2[p] = 0.0; S.L3[p] = 0.0;
            }
        }
        __syncthreads();
        for (int m = tid;; m += nth) {
            const int j = 2 * s - 1 + 2 * s * m;
            if (j >= n) break;
            const int p = j - s, q = j + s;
            double da = S.Da[j], db = S.Db[j], dc = S.Dc[j];
            double g0 = S.f0[j], g1 = S.f1[j];
            {   // lower neighbour p: coupling A = E_p (row p, col j)
                const double e0 = S.E0[p], e1 = S.E1[p], e2 = S.E2[p], e3 = S.E3[p];
                const double pa = S.Da[p], pb = S.Db[p], pc = S.Dc[p];
                const double t00 = e0 * pa + e2 * pb, t01 = e0 * pb + e2 * pc;
                const double t10 = e1 * pa + e3 * pb, t11 = e1 * pb + e3 * pc;
                da -= t00 * e0 + t01 * e2;
                db -= t00 * e1 + t01 * e3;
                dc -= t10 * e1 + t11 * e3;
                const double h0 = S.f0[p], h1 = S.f1[p];
                g0 -= t00 * h0 + t01 * h1;
                g1 -= t10 * h0 + t11 * h1;
            }
            double w = S.fw[j] - cup[p] * cinv[p] * S.fw[p];
            double n0 = 0.0, n1 = 0.0, n2 = 0.0, n3 = 0.0;
            if (q < n) {  // upper neighbour q: coupling A = E_j (row j, col q)
                const double e0 = S.E0[j], e1 = S.E1[j], e2 = S.E2[j], e3 = S.E3[j];
                const double qa = S.Da[q], qb = S.Db[q], qc = S.Dc[q];
                const double t00 = e0 * qa + e1 * qb, t01 = e0 * qb + e1 * qc;
                const double t10 = e2 * qa + e3 * qb, t11 = e2 * qb + e3 * qc;
                da -= t00 * e0 + t01 * e1;
                db -= t00 * e2 + t01 * e3;
                dc -= t10 * e2 + t11 * e3;
                const double h0 = S.f0[q], h1 = S.f1[q];
                g0 -= t00 * h0 + t01 * h1;
                g1 -= t10 * h0 + t11 * h1;
                if (q + s < n) {
                    const double k0 = S.E0[q], k1 = S.E1[q], k2 = S.E2[q], k3 = S.E3[q];
                    n0 = -(t00 * k0 + t01 * k2);
                    n1 = -(t00 * k1 + t01 * k3);
                    n2 = -(t10 * k0 + t11 * k2);
                    n3 = -(t10 * k1 + t11 * k3);
                }
                w -= clo[q] * cinv[q] * S.fw[q];
            }
            S.Da[j] = da; S.Db[j] = db; S.Dc[j] = dc;
            S.f0[j] = g0; S.f1[j] = g1;
            S.E0[j] = n0; S.E1[j] = n1; S.E2[j] = n2; S.E3[j] = n3;
            S.fw[j] = w;
        }
        __syncthreads();
    }
    if (tid == 0) {
        const int r = (1 << top) - 1;
        const double a = S.Da[r], b = S.Db[r], c = S.Dc[r];
        const double idet = 1.0 / (a * c - b * b);
        const double g0 = S.f0[r], g1 = S.f1[r];
        S.Da[r] = c * idet; S.Db[r] = -b * idet; S.Dc[r] = a * idet;
        S.f0[r] = (c * g0 - b * g1) * idet;
        S.f1[r] = (a * g1 - b * g0) * idet;
        S.fw[r] = cinv[r] * S.fw[r];
    }
    __syncthreads();
    for (int lev = top - 1; lev >= 0; --lev) {
        const int s = 1 << lev;
        for (int m = tid;; m += nth) {
            const int p = s - 1 + 2 * s * m;
            if (p >= n) break;
            double g0 = S.f0[p], g1 = S.f1[p], w = S.fw[p];
            if (p - s >= 0) {
                const double xa = S.f0[p - s], xb = S.f1[p - s];
                g0 -= S.L0[p] * xa + S.L2[p] * xb;
                g1 -= S.L1[p] * xa + S.L3[p] * xb;
                w -= clo[p] * S.fw[p - s];
            }
            if (p + s < n) {
                const double xa = S.f0[p + s], xb = S.f1[p + s];
                g0 -= S.E0[p] * xa + S.E1[p] * xb;
                g1 -= S.E2[p] * xa + S.E3[p] * xb;
                w -= cup[p] * S.fw[p + s];
            }
            const double pa = S.Da[p], pb = S.Db[p], pc = S.Dc[p];
            S.f0[p] = pa * g0 + pb * g1;
            S.f1[p] = pb * g0 + pc * g1;
            S.fw[p] = cinv[p] * w;
        }
        __syncthreads();
    }
}

// One block row: residual (or given rhs) -> exact local KKT solve -> update.
//   r = b - (D x + couplings(uprev, munext))   (x, uprev, munext may be null)
//   out = (xupd ? xupd : 0) + omega * D^{-1} r
// Pointers that may be written by the same kernel (serial substitution) are
// read through plain loads (no __restrict__/.nc).
__device__ void tri_block(const TView& V, int i, const double* b, const double* x,
                          const double* uprev, const double* munext, double* out, double omega,
                          const double* xupd, double* sm) {
    const Lay& L = V.lay;
    const int n = V.n;
    const int tid = threadIdx.x, nth = blockDim.x;
    const bool has_vm = i >= 1, has_uzl = i < L.N;
    TriSm S(sm, n);
    const double kap = V.kappa, k2 = kap * kap;
    const double* Qv = (i == L.N) ? V.Ql : V.Qm;
    const double* Qu = (i == L.N - 1) ? V.Ql : V.Qm;
    const double* Qz = V.Qz;
    const double* K = has_uzl ? V.K + (size_t)i * 3 * n : nullptr;
    const double* C = (has_uzl && has_vm) ? V.C + (size_t)i * 3 * n : nullptr;
    const int64_t ov = L.off_v(i), ou = L.off_u(i), oz = L.off_z(i), om = L.off_mu(i),
                  ol = L.off_l(i);

    for (int j = tid; j < n; j += nth) {
        double rv = 0.0, ru = 0.0, rz = 0.0, rm = 0.0, rl = 0.0;
        if (has_vm) { rv = b[ov + j]; rm = b[om + j]; }
        if (has_uzl) { ru = b[ou + j]; rz = b[oz + j]; rl = b[ol + j]; }
        if (x) {
            if (has_vm) {
                double av = tmv(Qv, n, x + ov, j) - x[om + j];
                if (C) av += tmtv(C, n, x + ol, j);
                rv -= av;
                rm += x[ov + j];
            }
            if (has_uzl) {
                ru -= tmv(Qu, n, x + ou, j) + tmtv(K, n, x + ol, j);
                rz -= tmv(Qz, n, x + oz, j) + kap * tmv(Qz, n, x + ol, j);
                double al = tmv(K, n, x + ou, j) + kap * tmv(Qz, n, x + oz, j);
                if (C) al += tmv(C, n, x + ov, j);
                rl -= al;
            }
        }
        if (has_vm && uprev) rm -= uprev[j];
        if (has_uzl && munext) ru -= munext[j];
        if (has_vm) { S.sv[j] = -rm; S.srv[j] = rv; }
        if (has_uzl) { S.f0[j] = ru; S.f1[j] = rl - kap * rz; S.fw[j] = rz; }
    }
    __syncthreads();
    if (!has_uzl) {  // last block (v_N, mu_N): mu = Qv v - r_v
        for (int j = tid; j < n; j += nth) {
            double dv = S.sv[j];
            double dm = tmv(Qv, n, S.sv, j) - S.srv[j];
            double bv = xupd ? xupd[ov + j] : 0.0, bm = xupd ? xupd[om + j] : 0.0;
            out[ov + j] = bv + omega * dv;
            out[om + j] = bm + omega * dm;
        }
        __syncthreads();
        return;
    }
    for (int j = tid; j < n; j += nth) {
        if (C) S.f1[j] -= tmv(C, n, S.sv, j);
        S.Da[j] = Qu[n + j];
        S.Db[j] = K[n + j];
        S.Dc[j] = -k2 * Qz[n + j];
        if (j < n - 1) {
            S.E0[j] = Qu[2 * n + j];
            S.E1[j] = K[j + 1];
            S.E2[j] = K[2 * n + j];
            S.E3[j] = -k2 * Qz[2 * n + j];
        } else {
            S.E0[j] = 0.0; S.E1[j] = 0.0; S.E2[j] = 0.0; S.E3[j] = 0.0;
        }
    }
    __syncthreads();
    cr_solve(n, S, V.cr);
    for (int j = tid; j < n; j += nth) {
        const double du = S.f0[j], dl = S.f1[j];
        const double dz = S.fw[j] - kap * dl;
        out[ou + j] = (xupd ? xupd[ou + j] : 0.0) + omega * du;
        out[oz + j] = (xupd ? xupd[oz + j] : 0.0) + omega * dz;
        out[ol + j] = (xupd ? xupd[ol + j] : 0.0) + omega * dl;
        if (has_vm) {
            const double dv = S.sv[j];
            double dm = tmv(Qv, n, S.sv, j) - S.srv[j];
            if (C) dm += tmtv(C, n, S.f1, j);
            out[ov + j] = (xupd ? xupd[ov + j] : 0.0) + omega * dv;
            out[om + j] = (xupd ? xupd[om + j] : 0.0) + omega * dm;
        }
    }
    __syncthreads();
}

// Parallel over block rows: jacobi (x may be null) or plain D^{-1} b.
__global__ void tri_rows(TView V, const double* __restrict__ b, const double* __restrict__ x,
                         double* __restrict__ y, double omega) {
    extern __shared__ double sm[];
    const Lay& L = V.lay;
    for (int i = blockIdx.x; i <= L.N; i += gridDim.x) {
        const double* uprev = (x && i >= 1) ? x + L.off_u(i - 1) : nullptr;
        const double* munext = (x && i < L.N) ? x + L.off_mu(i + 1) : nullptr;
        tri_block(V, i, b, x, uprev, munext, y, omega, x, sm);
    }
}

// Serial substitution over the time axis (smoothers.py:79-109), one CTA.
template <bool FORWARD>
__global__ void tri_subst(TView V, const double* __restrict__ r, double* d) {
    extern __shared__ double sm[];
    const Lay& L = V.lay;
    for (int k = 0; k <= L.N; ++k) {
        const int i = FORWARD ? k : L.N - k;
        const double* uprev = (FORWARD && i >= 1) ? d + L.off_u(i - 1) : nullptr;
        const double* munext = (!FORWARD && i < L.N) ? d + L.off_mu(i + 1) : nullptr;
        tri_block(V, i, r, nullptr, uprev, munext, d, 1.0, nullptr, sm);
    }
}

enum TriApply { T_APPLY = 0, T_APPLY_DIAG = 1, T_RESIDUAL = 2 };

// y = A x, D x, or b - A x; one CTA per block row, threads over nodes.
template <int MODE>
__global__ void tri_apply(TView V, const double* __restrict__ b, const double* __restrict__ x,
                          double* __restrict__ y) {
    const Lay& L = V.lay;
    const int n = V.n;
    const double kap = V.kappa;
    for (int i = blockIdx.x; i <= L.N; i += gridDim.x) {
        const bool has_vm = i >= 1, has_uzl = i < L.N;
        const double* Qv = (i == L.N) ? V.Ql : V.Qm;
        const double* Qu = (i == L.N - 1) ? V.Ql : V.Qm;
        const double* K = has_uzl ? V.K + (size_t)i * 3 * n : nullptr;
        const double* C = (has_uzl && has_vm) ? V.C + (size_t)i * 3 * n : nullptr;
        const int64_t ov = L.off_v(i), ou = L.off_u(i), oz = L.off_z(i), om = L.off_mu(i),
                      ol = L.off_l(i);
        const double* uprev = (MODE != T_APPLY_DIAG && has_vm) ? x + L.off_u(i - 1) : nullptr;
        const double* munext = (MODE != T_APPLY_DIAG && has_uzl) ? x + L.off_mu(i + 1) : nullptr;
        for (int j = threadIdx.x; j < n; j += blockDim.x) {
            if (has_vm) {
                double av = tmv(Qv, n, x + ov, j) - x[om + j];
                if (C) av += tmtv(C, n, x + ol, j);
                double am = -x[ov + j];
                if (uprev) am += uprev[j];
                if (MODE == T_RESIDUAL) { av = b[ov + j] - av; am = b[om + j] - am; }
                y[ov + j] = av;
                y[om + j] = am;
            }
            if (has_uzl) {
                double au = tmv(Qu, n, x + ou, j) + tmtv(K, n, x + ol, j);
                if (munext) au += munext[j];
                double az = tmv(V.Qz, n, x + oz, j) + kap * tmv(V.Qz, n, x + ol, j);
                double al = tmv(K, n, x + ou, j) + kap * tmv(V.Qz, n, x + oz, j);
                if (C) al += tmv(C, n, x + ov, j);
                if (MODE == T_RESIDUAL) {
                    au = b[ou + j] - au; az = b[oz + j] - az; al = b[ol + j] - al;
                }
                y[ou + j] = au;
                y[oz + j] = az;
                y[ol + j] = al;
            }
        }
    }
}

int64_t tri_smem_bytes(int n) {
    if (n < 2 || n > 1792) return 0;
    return (int64_t)kTriArrays * n * (int64_t)sizeof(double);
}

static int tri_threads(int n) {
    int t = (n / 2 + 31) / 32 * 32;
    if (t < 32) t = 32;
    if (t > 512) t = 512;
    return t;
}

int tri_launch(const tk_level* Lv, int op, const double* b, const double* x, double* y,
               double omega, cudaStream_t s) {
    TView V(Lv);
    const int n = Lv->n_u;
    if (Lv->n_z != Lv->n_u) {
        set_error("tri family needs n_z == n_u (got %d, %d)", Lv->n_u, Lv->n_z);
        return TK_ERR_UNSUPPORTED;
    }
    const int rows = Lv->n_steps + 1;
    if (op == T_APPLY || op == T_APPLY_DIAG || op == T_RESIDUAL) {
        const int th = n >= 256 ? 256 : 128;
        const int grid = rows < (1 << 30) ? rows : (1 << 30);
        if (op == T_APPLY) tri_apply<T_APPLY><<<grid, th, 0, s>>>(V, b, x, y);
        else if (op == T_APPLY_DIAG) tri_apply<T_APPLY_DIAG><<<grid, th, 0, s>>>(V, b, x, y);
        else tri_apply<T_RESIDUAL><<<grid, th, 0, s>>>(V, b, x, y);
        return check_launch("tri_apply");
    }
    const int64_t smem = tri_smem_bytes(n);
    if (smem == 0) {
        set_error("tri family kernels support 2 <= n_u <= 1792 (got %d)", n);
        return TK_ERR_UNSUPPORTED;
    }
    static bool attr_done = false;
    if (!attr_done) {
        cudaFuncSetAttribute(tri_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        cudaFuncSetAttribute(tri_subst<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             227 * 1024);
        cudaFuncSetAttribute(tri_subst<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             227 * 1024);
        attr_done = true;
    }
    const int th = tri_threads(n);
    switch (op) {
        case 3:  // diag solve
            tri_rows<<<rows, th, smem, s>>>(V, b, nullptr, y, 1.0);
            break;
        case 4:  // jacobi
            tri_rows<<<rows, th, smem, s>>>(V, b, x, y, omega);
            break;
        case 10: tri_subst<true><<<1, th, smem, s>>>(V, b, y); break;
        case 11: tri_subst<false><<<1, th, smem, s>>>(V, b, y); break;
        default: set_error("tri: bad op %d", op); return TK_ERR_ARG;
    }
    return check_launch("tri_rows");
}

}  // namespace tk
