// DENSE family: tiny per-interval KKT blocks (van der Pol: n_u = 2, n_z in {1,2}).
//
// One thread owns one block row of the Figure-3 operator (kkt.py:194-320);
// the local KKT solve is done in registers by eliminating (v, mu) exactly,
// then the control and the state through the constant weight inverses, and
// solving the n_u x n_u SPD Schur system
//     S = K Qu^{-1} K^T + B Qz^{-1} B^T
// for the dynamics multiplier.  This is D_i^{-1} of DiagonalSolver
// (kkt.py:338-389) without forming the (4nu+nz)^2 inverse: the HBM stream
// per interval is the vectors plus K_i, C_i, B_i only.
#include <stdlib.h>

#include "tk_common.cuh"

namespace tk {

template <int NU, int NZ>
struct DView {
    Lay lay;
    const double* __restrict__ K;
    const double* __restrict__ C;
    const double* __restrict__ B;
    const double* __restrict__ Qm;
    const double* __restrict__ Ql;
    const double* __restrict__ Qz;
    const double* __restrict__ Qm_inv;
    const double* __restrict__ Ql_inv;
    const double* __restrict__ Qz_inv;
    Slab sl;
    DView(const tk_level* L)
        : lay(L->n_steps, L->n_u, L->n_z), K(L->K), C(L->C), B(L->B), Qm(L->Qm), Ql(L->Ql),
          Qz(L->Qz), Qm_inv(L->Qm_inv), Ql_inv(L->Ql_inv), Qz_inv(L->Qz_inv),
          sl(L, Lay(L->n_steps, L->n_u, L->n_z)) {}
    // stage data of global block row i (stage arrays start at the slab's first row)
    __device__ const double* Ki(int i) const { return K + (size_t)(i - sl.r0) * NU * NU; }
    __device__ const double* Ci(int i) const { return C + (size_t)(i - sl.r0) * NU * NU; }
    __device__ const double* Bi(int i) const { return B + (size_t)(i - sl.r0) * NU * NZ; }
};

// y = A x, A row-major R x Cn
template <int R, int Cn>
__device__ __forceinline__ void mv(const double* __restrict__ A, const double* x, double* y) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < Cn; ++c) s += A[r * Cn + c] * x[c];
        y[r] = s;
    }
}
// y += A^T x, A row-major R x Cn (x length R, y length Cn)
template <int R, int Cn>
__device__ __forceinline__ void mtv_add(const double* __restrict__ A, const double* x, double* y) {
#pragma unroll
    for (int c = 0; c < Cn; ++c) {
        double s = 0.0;
#pragma unroll
        for (int r = 0; r < R; ++r) s += A[r * Cn + c] * x[r];
        y[c] += s;
    }
}
template <int R, int Cn>
__device__ __forceinline__ void mv_add(const double* __restrict__ A, const double* x, double* y) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < Cn; ++c) s += A[r * Cn + c] * x[c];
        y[r] += s;
    }
}

// Gaussian elimination with partial pivoting on a small dense system (in place).
template <int N>
__device__ __forceinline__ void small_solve(double (&A)[N][N], double (&b)[N]) {
#pragma unroll
    for (int k = 0; k < N; ++k) {
        int p = k;
        double best = fabs(A[k][k]);
#pragma unroll
        for (int r = k + 1; r < N; ++r) {
            double a = fabs(A[r][k]);
            if (a > best) { best = a; p = r; }
        }
        if (p != k) {
#pragma unroll
            for (int c = 0; c < N; ++c) {
                // unrolled swap with a runtime row index
#pragma unroll
                for (int r = k + 1; r < N; ++r)
                    if (r == p) { double t = A[k][c]; A[k][c] = A[r][c]; A[r][c] = t; }
            }
#pragma unroll
            for (int r = k + 1; r < N; ++r)
                if (r == p) { double t = b[k]; b[k] = b[r]; b[r] = t; }
        }
        double inv = 1.0 / A[k][k];
#pragma unroll
        for (int r = k + 1; r < N; ++r) {
            double l = A[r][k] * inv;
#pragma unroll
            for (int c = k + 1; c < N; ++c) A[r][c] -= l * A[k][c];
            b[r] -= l * b[k];
        }
    }
#pragma unroll
    for (int k = N - 1; k >= 0; --k) {
        double s = b[k];
#pragma unroll
        for (int c = k + 1; c < N; ++c) s -= A[k][c] * b[c];
        b[k] = s / A[k][k];
    }
}

template <int NU, int NZ>
struct Seg {
    double v[NU], u[NU], z[NZ], m[NU], l[NU];
};

template <int NU, int NZ>
__device__ __forceinline__ void load_seg(const Lay& lay, int i, const double* x, Seg<NU, NZ>& s,
                                         int64_t base = 0) {
#pragma unroll
    for (int e = 0; e < NU; ++e) { s.v[e] = 0.0; s.u[e] = 0.0; s.m[e] = 0.0; s.l[e] = 0.0; }
#pragma unroll
    for (int e = 0; e < NZ; ++e) s.z[e] = 0.0;
    if (x == nullptr) return;
    if (i >= 1) {
        const double* pv = x + (lay.off_v(i) - base);
        const double* pm = x + (lay.off_mu(i) - base);
#pragma unroll
        for (int e = 0; e < NU; ++e) { s.v[e] = pv[e]; s.m[e] = pm[e]; }
    }
    if (i < lay.N) {
        const double* pu = x + (lay.off_u(i) - base);
        const double* pz = x + (lay.off_z(i) - base);
        const double* pl = x + (lay.off_l(i) - base);
#pragma unroll
        for (int e = 0; e < NU; ++e) { s.u[e] = pu[e]; s.l[e] = pl[e]; }
#pragma unroll
        for (int e = 0; e < NZ; ++e) s.z[e] = pz[e];
    }
}

template <int NU, int NZ>
__device__ __forceinline__ void store_seg(const Lay& lay, int i, double* y, const Seg<NU, NZ>& s,
                                          int64_t base = 0) {
    if (i >= 1) {
        double* pv = y + (lay.off_v(i) - base);
        double* pm = y + (lay.off_mu(i) - base);
#pragma unroll
        for (int e = 0; e < NU; ++e) { pv[e] = s.v[e]; pm[e] = s.m[e]; }
    }
    if (i < lay.N) {
        double* pu = y + (lay.off_u(i) - base);
        double* pz = y + (lay.off_z(i) - base);
        double* pl = y + (lay.off_l(i) - base);
#pragma unroll
        for (int e = 0; e < NU; ++e) { pu[e] = s.u[e]; pl[e] = s.l[e]; }
#pragma unroll
        for (int e = 0; e < NZ; ++e) pz[e] = s.z[e];
    }
}

// (A x)_i with optional continuity couplings: uprev = u_i (from block i-1)
// feeding the mu rows, munext = mu_{i+1} (from block i+1) feeding the u rows.
template <int NU, int NZ>
__device__ __forceinline__ void apply_row(const DView<NU, NZ>& V, int i, const Seg<NU, NZ>& x,
                                          const double* uprev, const double* munext,
                                          Seg<NU, NZ>& y) {
    const Lay& L = V.lay;
    const bool has_vm = i >= 1, has_uzl = i < L.N;
#pragma unroll
    for (int e = 0; e < NU; ++e) { y.v[e] = 0.0; y.u[e] = 0.0; y.m[e] = 0.0; y.l[e] = 0.0; }
#pragma unroll
    for (int e = 0; e < NZ; ++e) y.z[e] = 0.0;
    if (has_vm) {
        const double* Qv = (i == L.N) ? V.Ql : V.Qm;  // q_v[i-1]
        mv<NU, NU>(Qv, x.v, y.v);
#pragma unroll
        for (int e = 0; e < NU; ++e) {
            y.v[e] -= x.m[e];
            y.m[e] = -x.v[e] + (uprev ? uprev[e] : 0.0);
        }
    }
    if (has_uzl) {
        const double* Qu = (i == L.N - 1) ? V.Ql : V.Qm;  // q_u[i]
        const double* K = V.Ki(i);
        const double* B = V.Bi(i);
        mv<NU, NU>(Qu, x.u, y.u);
        mtv_add<NU, NU>(K, x.l, y.u);
        if (munext) {
#pragma unroll
            for (int e = 0; e < NU; ++e) y.u[e] += munext[e];
        }
        mv<NZ, NZ>(V.Qz, x.z, y.z);
        mtv_add<NU, NZ>(B, x.l, y.z);
        mv<NU, NU>(K, x.u, y.l);
        mv_add<NU, NZ>(B, x.z, y.l);
        if (has_vm) {
            const double* C = V.Ci(i);
            mtv_add<NU, NU>(C, x.l, y.v);
            mv_add<NU, NU>(C, x.v, y.l);
        }
    }
}

// d = D_i^{-1} r (local KKT solve of block row i).
template <int NU, int NZ>
__device__ __forceinline__ void solve_row(const DView<NU, NZ>& V, int i, const Seg<NU, NZ>& r,
                                          Seg<NU, NZ>& d) {
    const Lay& L = V.lay;
    const bool has_vm = i >= 1, has_uzl = i < L.N;
    double rl[NU];
#pragma unroll
    for (int e = 0; e < NU; ++e) rl[e] = r.l[e];
    if (has_vm) {
#pragma unroll
        for (int e = 0; e < NU; ++e) d.v[e] = -r.m[e];  // mu-row: -v = r_mu
    }
    if (has_uzl) {
        const double* Qu_inv = (i == L.N - 1) ? V.Ql_inv : V.Qm_inv;
        const double* K = V.Ki(i);
        const double* B = V.Bi(i);
        if (has_vm) {
            const double* C = V.Ci(i);
            double cv[NU];
            mv<NU, NU>(C, d.v, cv);
#pragma unroll
            for (int e = 0; e < NU; ++e) rl[e] -= cv[e];
        }
        // a = Qu^{-1} r_u, c = Qz^{-1} r_z
        double a[NU], c[NZ];
        mv<NU, NU>(Qu_inv, r.u, a);
        mv<NZ, NZ>(V.Qz_inv, r.z, c);
        // S = K Qu^-1 K^T + B Qz^-1 B^T ; t = K a + B c - rl
        double KQ[NU][NU], BQ[NU][NZ];
#pragma unroll
        for (int p = 0; p < NU; ++p) {
#pragma unroll
            for (int q = 0; q < NU; ++q) {
                double s = 0.0;
#pragma unroll
                for (int k = 0; k < NU; ++k) s += K[p * NU + k] * Qu_inv[k * NU + q];
                KQ[p][q] = s;
            }
#pragma unroll
            for (int q = 0; q < NZ; ++q) {
                double s = 0.0;
#pragma unroll
                for (int k = 0; k < NZ; ++k) s += B[p * NZ + k] * V.Qz_inv[k * NZ + q];
                BQ[p][q] = s;
            }
        }
        double S[NU][NU], t[NU];
#pragma unroll
        for (int p = 0; p < NU; ++p) {
#pragma unroll
            for (int q = 0; q < NU; ++q) {
                double s = 0.0;
#pragma unroll
                for (int k = 0; k < NU; ++k) s += KQ[p][k] * K[q * NU + k];
#pragma unroll
                for (int k = 0; k < NZ; ++k) s += BQ[p][k] * B[q * NZ + k];
                S[p][q] = s;
            }
            double s = -rl[p];
#pragma unroll
            for (int k = 0; k < NU; ++k) s += K[p * NU + k] * a[k];
#pragma unroll
            for (int k = 0; k < NZ; ++k) s += B[p * NZ + k] * c[k];
            t[p] = s;
        }
        small_solve<NU>(S, t);
#pragma unroll
        for (int e = 0; e < NU; ++e) d.l[e] = t[e];
        // u = Qu^{-1}(r_u - K^T lam), z = Qz^{-1}(r_z - B^T lam)
        double ku[NU], bz[NZ];
#pragma unroll
        for (int e = 0; e < NU; ++e) ku[e] = r.u[e];
#pragma unroll
        for (int e = 0; e < NZ; ++e) bz[e] = r.z[e];
#pragma unroll
        for (int q = 0; q < NU; ++q) {
#pragma unroll
            for (int p = 0; p < NU; ++p) ku[q] -= K[p * NU + q] * t[p];
        }
#pragma unroll
        for (int q = 0; q < NZ; ++q) {
#pragma unroll
            for (int p = 0; p < NU; ++p) bz[q] -= B[p * NZ + q] * t[p];
        }
        mv<NU, NU>(Qu_inv, ku, d.u);
        mv<NZ, NZ>(V.Qz_inv, bz, d.z);
    }
    if (has_vm) {
        // v-row: Qv v - mu + C^T lam = r_v  =>  mu = Qv v + C^T lam - r_v
        const double* Qv = (i == L.N) ? V.Ql : V.Qm;
        mv<NU, NU>(Qv, d.v, d.m);
        if (has_uzl) {
            const double* C = V.Ci(i);
            mtv_add<NU, NU>(C, d.l, d.m);
        }
#pragma unroll
        for (int e = 0; e < NU; ++e) d.m[e] -= r.v[e];
    }
}

enum DenseMode { D_APPLY = 0, D_APPLY_DIAG = 1, D_RESIDUAL = 2, D_SOLVE = 3, D_JACOBI = 4 };

// rc != nullptr (D_JACOBI, x == nullptr, omega == 1, whole level, even N): the
// zero-start sweep also writes the restricted residual of
// tk_residual_restrict_jacobi0 (row 2c-1: coarse mu_c = -u_{2c}; row 2c:
// coarse u_c = -mu_{2c} and the zero v_c, z_{c+1}, lam_{c+1} of coarse row c).
template <int NU, int NZ, int MODE>
__global__ void __launch_bounds__(128) dense_rows(DView<NU, NZ> V, const double* __restrict__ b,
                                                  const double* __restrict__ x,
                                                  double* __restrict__ y, double omega,
                                                  double* __restrict__ rc = nullptr) {
    const Lay& L = V.lay;
    const Slab& S = V.sl;
    const int64_t bs0 = S.base;
    for (int i = S.r0 + blockIdx.x * blockDim.x + threadIdx.x; i < S.r1;
         i += gridDim.x * blockDim.x) {
        Seg<NU, NZ> xs, ys;
        const double* uprev = x ? S.uprev(L, x, i) : nullptr;
        const double* munext = x ? S.munext(L, x, i) : nullptr;
        if (MODE == D_SOLVE) {
            load_seg<NU, NZ>(L, i, b, xs, bs0);
            solve_row<NU, NZ>(V, i, xs, ys);
            store_seg<NU, NZ>(L, i, y, ys, bs0);
            continue;
        }
        load_seg<NU, NZ>(L, i, x, xs, bs0);
        apply_row<NU, NZ>(V, i, xs, MODE == D_APPLY_DIAG ? nullptr : uprev,
                          MODE == D_APPLY_DIAG ? nullptr : munext, ys);
        if (MODE == D_APPLY || MODE == D_APPLY_DIAG) {
            store_seg<NU, NZ>(L, i, y, ys, bs0);
            continue;
        }
        Seg<NU, NZ> bs;
        load_seg<NU, NZ>(L, i, b, bs, bs0);
#pragma unroll
        for (int e = 0; e < NU; ++e) {
            bs.v[e] -= ys.v[e]; bs.u[e] -= ys.u[e]; bs.m[e] -= ys.m[e]; bs.l[e] -= ys.l[e];
        }
#pragma unroll
        for (int e = 0; e < NZ; ++e) bs.z[e] -= ys.z[e];
        if (MODE == D_RESIDUAL) {
            store_seg<NU, NZ>(L, i, y, bs, bs0);
            continue;
        }
        // D_JACOBI: x_out = x + omega * D^{-1} (b - A x)
        solve_row<NU, NZ>(V, i, bs, ys);
#pragma unroll
        for (int e = 0; e < NU; ++e) {
            xs.v[e] += omega * ys.v[e]; xs.u[e] += omega * ys.u[e];
            xs.m[e] += omega * ys.m[e]; xs.l[e] += omega * ys.l[e];
        }
#pragma unroll
        for (int e = 0; e < NZ; ++e) xs.z[e] += omega * ys.z[e];
        store_seg<NU, NZ>(L, i, y, xs, bs0);
        if (MODE == D_JACOBI && rc) {
            const Lay Lc(L.N / 2, NU, NZ);
            if (i & 1) {
                double* p = rc + Lc.t_mu((i + 1) / 2);
#pragma unroll
                for (int e = 0; e < NU; ++e) p[e] = 0.0 - xs.u[e];
            } else {
                const int c = i / 2;
                if (i >= 2) {
                    double* p = rc + Lc.t_u(c);
#pragma unroll
                    for (int e = 0; e < NU; ++e) p[e] = 0.0 - xs.m[e];
                }
                if (c >= 1) {
                    double* p = rc + Lc.off_v(c);
#pragma unroll
                    for (int e = 0; e < NU; ++e) p[e] = 0.0;
                }
                if (c < Lc.N) {
                    double* pz = rc + Lc.off_z(c);
                    double* pl = rc + Lc.off_l(c);
#pragma unroll
                    for (int e = 0; e < NZ; ++e) pz[e] = 0.0;
#pragma unroll
                    for (int e = 0; e < NU; ++e) pl[e] = 0.0;
                }
            }
        }
    }
}


// Splitting-form rows (omega = 1 or from zero; the DENSE twin of
// tri_rows_part<.., 3, ..>): y = D^{-1}(b + (L + U) x) -- the local solve of b
// with the continuity couplings u_{i-1}, mu_{i+1} of x moved to the
// right-hand side, so x is read at those two segments only.
//   ec != nullptr: the couplings are those of x + P ec (the V-cycle's
//     prolongation folded into the post-smoothing sweep, multigrid.py:115-132,
//     :297-299; the arithmetic of tk_prolong_add);
//   rc != nullptr (x == nullptr, whole level, even N): the zero-start sweep
//     also writes its restricted residual (as dense_rows<.., D_JACOBI> does);
//     partial: only the u and mu segments of y are stored.
template <int NU, int NZ>
__global__ void __launch_bounds__(128) dense_rows_split(DView<NU, NZ> V, const double* __restrict__ b,
                                                        const double* __restrict__ x,
                                                        double* __restrict__ y, double omega,
                                                        const double* __restrict__ ec,
                                                        double* __restrict__ rc, int partial,
                                                        const double* __restrict__ chalo) {
    const Lay& L = V.lay;
    const Slab& S = V.sl;
    const int64_t bs0 = S.base;
    const Lay Lc(L.N / 2, NU, NZ);
    // time slab: coarse rows [c0, c1) stored from offset cb; coarse segments
    // outside the slab come from chalo = [prev (u, lam) | next (v, mu)], the two
    // coarse entries fed by the neighbours' rows from tk_restrict_fix_slab
    const int c0 = S.r0 / 2, c1 = S.r1 == L.N + 1 ? L.N / 2 + 1 : S.r1 / 2;
    const int64_t cb = Lc.start(c0);
    auto cu = [&](int tc) -> const double* {
        return tc - 1 >= c0 ? ec + (Lc.t_u(tc) - cb) : chalo;
    };
    auto cm = [&](int tc) -> const double* {
        return tc < c1 ? ec + (Lc.t_mu(tc) - cb) : chalo + 3 * NU;
    };
    for (int i = S.r0 + blockIdx.x * blockDim.x + threadIdx.x; i < S.r1;
         i += gridDim.x * blockDim.x) {
        Seg<NU, NZ> bs, ys;
        load_seg<NU, NZ>(L, i, b, bs, bs0);
        const double* uprev = x ? S.uprev(L, x, i) : nullptr;
        const double* munext = x ? S.munext(L, x, i) : nullptr;
        if (uprev) {          // u_t, t = i
            const int t = i;
            const double* ca = nullptr;
            const double* cb2 = nullptr;
            if (ec) {
                if ((t & 1) == 0 || t == 1) ca = cu(t == 1 ? 1 : t / 2);
                else { ca = cu((t - 1) / 2); cb2 = cu((t + 1) / 2); }
            }
#pragma unroll
            for (int e = 0; e < NU; ++e) {
                double up = uprev[e];
                if (ca) up = cb2 ? up + 0.5 * (ca[e] + cb2[e]) : up + ca[e];
                bs.m[e] -= up;
            }
        }
        if (munext) {         // mu_t, t = i + 1
            const int t = i + 1;
            const double* ca = nullptr;
            const double* cb2 = nullptr;
            if (ec) {
                if ((t & 1) == 0 || t == 1) ca = cm(t == 1 ? 1 : t / 2);
                else { ca = cm((t - 1) / 2); cb2 = cm((t + 1) / 2); }
            }
#pragma unroll
            for (int e = 0; e < NU; ++e) {
                double mn = munext[e];
                if (ca) mn = cb2 ? mn + 0.5 * (ca[e] + cb2[e]) : mn + ca[e];
                bs.u[e] -= mn;
            }
        }
        solve_row<NU, NZ>(V, i, bs, ys);
#pragma unroll
        for (int e = 0; e < NU; ++e) {
            ys.v[e] = 0.0 + omega * ys.v[e]; ys.u[e] = 0.0 + omega * ys.u[e];
            ys.m[e] = 0.0 + omega * ys.m[e]; ys.l[e] = 0.0 + omega * ys.l[e];
        }
#pragma unroll
        for (int e = 0; e < NZ; ++e) ys.z[e] = 0.0 + omega * ys.z[e];
        if (partial) {
            if (i >= 1) {
                double* pm = y + (L.off_mu(i) - bs0);
#pragma unroll
                for (int e = 0; e < NU; ++e) pm[e] = ys.m[e];
            }
            if (i < L.N) {
                double* pu = y + (L.off_u(i) - bs0);
#pragma unroll
                for (int e = 0; e < NU; ++e) pu[e] = ys.u[e];
            }
        } else {
            store_seg<NU, NZ>(L, i, y, ys, bs0);
        }
        if (rc) {   // R (b - A y) = R (L + U)(y - x): couplings of the update
            if (i & 1) {
                if ((i + 1) / 2 < c1) {
                    double* p = rc + (Lc.t_mu((i + 1) / 2) - cb);
                    const double* xo = x ? x + (L.off_u(i) - bs0) : nullptr;
#pragma unroll
                    for (int e = 0; e < NU; ++e) p[e] = (xo ? xo[e] : 0.0) - ys.u[e];
                }
            } else {
                const int c = i / 2;
                if (i >= 2 && c - 1 >= c0) {
                    double* p = rc + (Lc.t_u(c) - cb);
                    const double* xo = x ? x + (L.off_mu(i) - bs0) : nullptr;
#pragma unroll
                    for (int e = 0; e < NU; ++e) p[e] = (xo ? xo[e] : 0.0) - ys.m[e];
                }
                if (c >= 1) {
                    double* p = rc + (Lc.off_v(c) - cb);
#pragma unroll
                    for (int e = 0; e < NU; ++e) p[e] = 0.0;
                }
                if (c < Lc.N) {
                    double* pz = rc + (Lc.off_z(c) - cb);
                    double* pl = rc + (Lc.off_l(c) - cb);
#pragma unroll
                    for (int e = 0; e < NZ; ++e) pz[e] = 0.0;
#pragma unroll
                    for (int e = 0; e < NU; ++e) pl[e] = 0.0;
                }
            }
        }
    }
}

template <int NU, int NZ>
static int dense_split_t(const tk_level* Lv, const double* b, const double* x, double* y,
                         double omega, const double* ec, double* rc, int partial, cudaStream_t s,
                         const double* chalo) {
    DView<NU, NZ> V(Lv);
    const int rows = V.sl.r1 - V.sl.r0;
    dense_rows_split<NU, NZ><<<grid_for(rows, 128, 1 << 20), 128, 0, s>>>(V, b, x, y, omega, ec, rc,
                                                                           partial, chalo);
    return check_launch("dense_rows_split");
}

template <int NU, int NZ>
static int dense_jacobi0_restrict_t(const tk_level* Lv, const double* b, double* y, double* rc,
                                    cudaStream_t s) {
    DView<NU, NZ> V(Lv);
    const int rows = V.sl.r1 - V.sl.r0;
    dense_rows<NU, NZ, D_JACOBI><<<grid_for(rows, 128, 1 << 20), 128, 0, s>>>(V, b, nullptr, y, 1.0, rc);
    return check_launch("dense_rows (jacobi0 + restrict)");
}

// Serial block substitution (smoothers.py:79-109): one thread walks the time axis.
template <int NU, int NZ, bool FORWARD>
__global__ void dense_subst(DView<NU, NZ> V, const double* __restrict__ r, double* __restrict__ d) {
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    const Lay& L = V.lay;
    for (int k = 0; k <= L.N; ++k) {
        const int i = FORWARD ? k : L.N - k;
        Seg<NU, NZ> rs, ds;
        load_seg<NU, NZ>(L, i, r, rs);
        if (FORWARD && i >= 1) {
            const volatile double* up = d + L.off_u(i - 1);
#pragma unroll
            for (int e = 0; e < NU; ++e) rs.m[e] -= up[e];
        }
        if (!FORWARD && i < L.N) {
            const volatile double* mn = d + L.off_mu(i + 1);
#pragma unroll
            for (int e = 0; e < NU; ++e) rs.u[e] -= mn[e];
        }
        solve_row<NU, NZ>(V, i, rs, ds);
        store_seg<NU, NZ>(L, i, d, ds);
    }
}

// ---------------------------------------------------------------------------
// Gauss-Seidel substitution as parallel solve -> chain -> parallel solve.
// Forward: u_i = a_i^u - G_i u_{i-1} with G_i = P_u D_i^{-1} E_mu; backward:
// mu_i = a_i^mu - H_i mu_{i+1} with H_i = P_mu D_i^{-1} E_u (nu x nu, built
// once by dense_factor).  The affine chain is evaluated by one CTA as a
// chunked parallel scan of map compositions.
// ---------------------------------------------------------------------------
template <int NU, int NZ>
__global__ void dense_factor(DView<NU, NZ> V, double* __restrict__ fac) {
    const Lay& L = V.lay;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= L.N; i += gridDim.x * blockDim.x) {
        double* G = fac + (size_t)i * 2 * NU * NU;
        double* H = G + NU * NU;
        for (int e = 0; e < 2 * NU * NU; ++e) G[e] = 0.0;
        if (i == 0 || i == L.N) continue;
#pragma unroll
        for (int k = 0; k < NU; ++k) {
            Seg<NU, NZ> r, d;
            load_seg<NU, NZ>(L, i, nullptr, r);
            r.m[k] = 1.0;
            solve_row<NU, NZ>(V, i, r, d);
#pragma unroll
            for (int e = 0; e < NU; ++e) G[e * NU + k] = d.u[e];
            load_seg<NU, NZ>(L, i, nullptr, r);
            r.u[k] = 1.0;
            solve_row<NU, NZ>(V, i, r, d);
#pragma unroll
            for (int e = 0; e < NU; ++e) H[e * NU + k] = d.m[e];
        }
    }
}

template <int NU>
struct Aff {  // x -> P x + p
    double P[NU][NU];
    double p[NU];
};

template <int NU>
__device__ __forceinline__ void aff_compose(const Aff<NU>& second, const Aff<NU>& first,
                                            Aff<NU>& out) {
#pragma unroll
    for (int r = 0; r < NU; ++r) {
        double s = second.p[r];
#pragma unroll
        for (int c = 0; c < NU; ++c) {
            double t = 0.0;
#pragma unroll
            for (int k = 0; k < NU; ++k) t += second.P[r][k] * first.P[k][c];
            out.P[r][c] = t;
            s += second.P[r][c] * first.p[c];
        }
        out.p[r] = s;
    }
}

template <int NU>
struct ScanT { static constexpr int value = NU <= 2 ? 256 : 64; };

template <int NU, bool FWD>
__global__ void __launch_bounds__(ScanT<NU>::value) dense_chain(Lay L, const double* __restrict__ a,
                                                            const double* __restrict__ fac,
                                                            double* __restrict__ chain) {
    constexpr int kScanThreads = ScanT<NU>::value;
    __shared__ Aff<NU> maps[2][kScanThreads];
    const int N = L.N, tid = threadIdx.x;
    const int M = N - 1;
    const int c = (M + kScanThreads - 1) / kScanThreads;
    const int lo = tid * c, hi = min(M, lo + c);
    auto blk = [&](int k) { return FWD ? 1 + k : N - 1 - k; };
    auto aseg = [&](int i) { return a + (FWD ? L.off_u(i) : L.off_mu(i)); };
    auto mat = [&](int i) { return fac + (size_t)i * 2 * NU * NU + (FWD ? 0 : NU * NU); };
    double x0[NU];
    {
        const double* s0 = aseg(FWD ? 0 : N);
#pragma unroll
        for (int e = 0; e < NU; ++e) x0[e] = s0[e];
        if (tid == 0) {
#pragma unroll
            for (int e = 0; e < NU; ++e) chain[(size_t)(FWD ? 0 : N) * NU + e] = x0[e];
        }
    }
    Aff<NU> F;
#pragma unroll
    for (int r = 0; r < NU; ++r) {
        F.p[r] = 0.0;
#pragma unroll
        for (int q = 0; q < NU; ++q) F.P[r][q] = (r == q) ? 1.0 : 0.0;
    }
    for (int k = lo; k < hi; ++k) {   // F <- (x -> a - G x) o F
        const int i = blk(k);
        const double* G = mat(i);
        const double* ai = aseg(i);
        Aff<NU> S, T;
#pragma unroll
        for (int r = 0; r < NU; ++r) {
            S.p[r] = ai[r];
#pragma unroll
            for (int q = 0; q < NU; ++q) S.P[r][q] = -G[r * NU + q];
        }
        aff_compose<NU>(S, F, T);
        F = T;
    }
    maps[0][tid] = F;
    __syncthreads();
    int src = 0;
    for (int d = 1; d < kScanThreads; d <<= 1) {   // inclusive Hillis-Steele scan
        if (tid >= d) aff_compose<NU>(maps[src][tid], maps[src][tid - d], maps[src ^ 1][tid]);
        else maps[src ^ 1][tid] = maps[src][tid];
        src ^= 1;
        __syncthreads();
    }
    double x[NU];
    if (tid == 0) {
#pragma unroll
        for (int e = 0; e < NU; ++e) x[e] = x0[e];
    } else {
        const Aff<NU>& S = maps[src][tid - 1];
#pragma unroll
        for (int r = 0; r < NU; ++r) {
            double s = S.p[r];
#pragma unroll
            for (int q = 0; q < NU; ++q) s += S.P[r][q] * x0[q];
            x[r] = s;
        }
    }
    for (int k = lo; k < hi; ++k) {
        const int i = blk(k);
        const double* G = mat(i);
        const double* ai = aseg(i);
        double y[NU];
#pragma unroll
        for (int r = 0; r < NU; ++r) {
            double s = ai[r];
#pragma unroll
            for (int q = 0; q < NU; ++q) s -= G[r * NU + q] * x[q];
            y[r] = s;
        }
#pragma unroll
        for (int r = 0; r < NU; ++r) {
            x[r] = y[r];
            chain[(size_t)i * NU + r] = y[r];
        }
    }
}

template <int NU, int NZ, bool FWD>
__global__ void __launch_bounds__(128) dense_rows_cpl(DView<NU, NZ> V, const double* __restrict__ r,
                                                      const double* __restrict__ chain,
                                                      double* __restrict__ y) {
    const Lay& L = V.lay;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= L.N; i += gridDim.x * blockDim.x) {
        Seg<NU, NZ> rs, ds;
        load_seg<NU, NZ>(L, i, r, rs);
        if (FWD && i >= 1) {
#pragma unroll
            for (int e = 0; e < NU; ++e) rs.m[e] -= chain[(size_t)(i - 1) * NU + e];
        }
        if (!FWD && i < L.N) {
#pragma unroll
            for (int e = 0; e < NU; ++e) rs.u[e] -= chain[(size_t)(i + 1) * NU + e];
        }
        solve_row<NU, NZ>(V, i, rs, ds);
        store_seg<NU, NZ>(L, i, y, ds);
    }
}

int64_t dense_fac_len(const tk_level* Lv) {
    return (int64_t)(Lv->n_steps + 1) * 2 * Lv->n_u * Lv->n_u;
}
int64_t dense_scratch_len(const tk_level* Lv) { return (int64_t)(Lv->n_steps + 1) * Lv->n_u; }

static bool dense_resid_form() {
    static const bool on = [] {
        const char* e = getenv("TK_JACOBI_RESIDUAL_FORM");
        return e && e[0] == '1';
    }();
    return on;
}

template <int NU, int NZ>
static int dense_launch_t(const tk_level* Lv, int op, const double* b, const double* x, double* y,
                          double omega, cudaStream_t s) {
    DView<NU, NZ> V(Lv);
    const int rows = V.sl.r1 - V.sl.r0;
    const int th = 128;
    const int grid = grid_for(rows, th, 1 << 20);
    if (op >= 10 && !V.sl.whole(Lv->n_steps)) {
        set_error("block Gauss-Seidel substitution needs the whole level (no time slab)");
        return TK_ERR_ARG;
    }
    switch (op) {
        case D_APPLY: dense_rows<NU, NZ, D_APPLY><<<grid, th, 0, s>>>(V, b, x, y, omega); break;
        case D_APPLY_DIAG:
            dense_rows<NU, NZ, D_APPLY_DIAG><<<grid, th, 0, s>>>(V, b, x, y, omega); break;
        case D_RESIDUAL: dense_rows<NU, NZ, D_RESIDUAL><<<grid, th, 0, s>>>(V, b, x, y, omega); break;
        case D_SOLVE: dense_rows<NU, NZ, D_SOLVE><<<grid, th, 0, s>>>(V, b, x, y, omega); break;
        case D_JACOBI:
            // omega = 1 or from zero: x enters through the two couplings only
            // (TK_JACOBI_RESIDUAL_FORM=1 keeps x + omega D^{-1}(b - A x))
            if ((x == nullptr || omega == 1.0) && !dense_resid_form())
                return dense_split_t<NU, NZ>(Lv, b, x, y, omega, nullptr, nullptr, 0, s, nullptr);
            dense_rows<NU, NZ, D_JACOBI><<<grid, th, 0, s>>>(V, b, x, y, omega);
            break;
        case 10:
        case 11: {
            const bool fwd = op == 10;
            if (!Lv->fac || !Lv->scratch) {
                if (fwd) dense_subst<NU, NZ, true><<<1, 1, 0, s>>>(V, b, y);
                else dense_subst<NU, NZ, false><<<1, 1, 0, s>>>(V, b, y);
                break;
            }
            dense_rows<NU, NZ, D_SOLVE><<<grid, th, 0, s>>>(V, b, nullptr, y, 1.0);
            if (fwd) {
                dense_chain<NU, true><<<1, ScanT<NU>::value, 0, s>>>(V.lay, y, Lv->fac, Lv->scratch);
                dense_rows_cpl<NU, NZ, true><<<grid, th, 0, s>>>(V, b, Lv->scratch, y);
            } else {
                dense_chain<NU, false><<<1, ScanT<NU>::value, 0, s>>>(V.lay, y, Lv->fac, Lv->scratch);
                dense_rows_cpl<NU, NZ, false><<<grid, th, 0, s>>>(V, b, Lv->scratch, y);
            }
            break;
        }
        case 12:
            if (!Lv->fac) { set_error("tk_subst_factor: level has no fac buffer"); return TK_ERR_ARG; }
            dense_factor<NU, NZ><<<grid, th, 0, s>>>(V, Lv->fac);
            break;
        default: set_error("dense: bad op %d", op); return TK_ERR_ARG;
    }
    return check_launch("dense_rows");
}

#define TK_DENSE_NZ(NU)                                                               \
    switch (Lv->n_z) {                                                                \
        case 1: return dense_launch_t<NU, 1>(Lv, op, b, x, y, omega, s);              \
        case 2: return dense_launch_t<NU, 2>(Lv, op, b, x, y, omega, s);              \
        case 3: return dense_launch_t<NU, 3>(Lv, op, b, x, y, omega, s);              \
        case 4: return dense_launch_t<NU, 4>(Lv, op, b, x, y, omega, s);              \
        default: break;                                                               \
    }

int dense_jacobi0_restrict(const tk_level* Lv, const double* b, double* y, double* rc,
                           cudaStream_t s) {
#define TK_DJR(NU, NZ) \
    if (Lv->n_u == NU && Lv->n_z == NZ) return dense_jacobi0_restrict_t<NU, NZ>(Lv, b, y, rc, s);
    TK_DJR(1, 1) TK_DJR(1, 2) TK_DJR(1, 3) TK_DJR(1, 4)
    TK_DJR(2, 1) TK_DJR(2, 2) TK_DJR(2, 3) TK_DJR(2, 4)
    TK_DJR(3, 1) TK_DJR(3, 2) TK_DJR(3, 3) TK_DJR(3, 4)
    TK_DJR(4, 1) TK_DJR(4, 2) TK_DJR(4, 3) TK_DJR(4, 4)
#undef TK_DJR
    set_error("dense family supports 1<=n_u,n_z<=4 (got n_u=%d n_z=%d)", Lv->n_u, Lv->n_z);
    return TK_ERR_UNSUPPORTED;
}

// tk_jacobi0_restrict_um (x == nullptr, rc, partial) / tk_jacobi_prolong (x, ec) on DENSE levels
int dense_split(const tk_level* Lv, const double* b, const double* x, double* y, const double* ec,
                double* rc, int partial, cudaStream_t s, const double* chalo) {
#define TK_DSP(NU, NZ) \
    if (Lv->n_u == NU && Lv->n_z == NZ) return dense_split_t<NU, NZ>(Lv, b, x, y, 1.0, ec, rc, partial, s, chalo);
    TK_DSP(1, 1) TK_DSP(1, 2) TK_DSP(1, 3) TK_DSP(1, 4)
    TK_DSP(2, 1) TK_DSP(2, 2) TK_DSP(2, 3) TK_DSP(2, 4)
    TK_DSP(3, 1) TK_DSP(3, 2) TK_DSP(3, 3) TK_DSP(3, 4)
    TK_DSP(4, 1) TK_DSP(4, 2) TK_DSP(4, 3) TK_DSP(4, 4)
#undef TK_DSP
    set_error("dense family supports 1<=n_u,n_z<=4 (got n_u=%d n_z=%d)", Lv->n_u, Lv->n_z);
    return TK_ERR_UNSUPPORTED;
}

int denseg_launch(const tk_level* Lv, int op, const double* b, const double* x, double* y,
                  double omega, cudaStream_t s);

int dense_launch(const tk_level* Lv, int op, const double* b, const double* x, double* y,
                 double omega, cudaStream_t s) {
    if (Lv->n_u > TK_MAX_DENSE || Lv->n_z > TK_MAX_DENSE)   // general sizes: tk_denseg.cu
        return denseg_launch(Lv, op, b, x, y, omega, s);
    switch (Lv->n_u) {
        case 1: TK_DENSE_NZ(1); break;
        case 2: TK_DENSE_NZ(2); break;
        case 3: TK_DENSE_NZ(3); break;
        case 4: TK_DENSE_NZ(4); break;
        default: break;
    }
    set_error("dense family supports 1<=n_u,n_z<=4 (got n_u=%d n_z=%d)", Lv->n_u, Lv->n_z);
    return TK_ERR_UNSUPPORTED;
}

}  // namespace tk
