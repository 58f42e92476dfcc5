// TRI family: per-interval KKT blocks whose sub-blocks are tridiagonal in
// space (P1 finite elements, 1D Burgers: problems.py:149-197).
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
// no pivoting.  All reductions run in shared memory; node j lives at the
// padded index PI(j) = j + j/16, which keeps every stride-2^l reduction
// level free of (or at most 2-way) bank conflicts.
//
// Every kernel is templated on NT, the number of spatial nodes when it is a
// compile-time constant (64..2048 are dispatched; NT = 0 is the generic
// runtime-n build): shared-memory row offsets then fold into immediates and
// the cyclic-reduction level loops unroll.
#include "tk_tri.cuh"

#include <cooperative_groups.h>
#include <math.h>
#include <string.h>

namespace cg = cooperative_groups;

namespace tk {

static constexpr int kMaxLev = 12;   // n <= 4096

static constexpr int kFacRows = 14;

// Cut level c of the chain's cyclic reduction: levels below c run as usual;
// the reduced system on the A = n >> c <= 32 active nodes left at level c is
// solved with its precomputed dense inverse W (2A x 2A, stored transposed).
#ifndef TK_CUT_A
#define TK_CUT_A 32   // largest reduced system solved densely (nodes)
#endif
__host__ __device__ __forceinline__ constexpr int cut_level(int n) {
    int c = 0;
    while ((n >> c) > TK_CUT_A) ++c;
    return c;
}
__host__ __device__ __forceinline__ constexpr int cut_nodes(int n) { return n >> cut_level(n); }
// doubles per interval record: P, M1, M2 (levels < c, level order), C, W^T
__host__ __device__ __forceinline__ constexpr int fac_record(int n) {
    return kFacRows * n + 4 * cut_nodes(n) * cut_nodes(n);
}


static constexpr int kTriArrays = 16;

// 16 padded node arrays; all addressed from one base with constant row offsets
// when n is a compile-time constant.
struct TriSm {
    double* b;
    int np;
    __device__ TriSm(double* sm, int n) : b(sm), np(padded(n)) {}
    __device__ double* Da() const { return b; }
    __device__ double* Db() const { return b + np; }
    __device__ double* Dc() const { return b + 2 * np; }
    __device__ double* E0() const { return b + 3 * np; }
    __device__ double* E1() const { return b + 4 * np; }
    __device__ double* E2() const { return b + 5 * np; }
    __device__ double* E3() const { return b + 6 * np; }
    __device__ double* L0() const { return b + 7 * np; }
    __device__ double* L1() const { return b + 8 * np; }
    __device__ double* L2() const { return b + 9 * np; }
    __device__ double* L3() const { return b + 10 * np; }
    __device__ double* f0() const { return b + 11 * np; }
    __device__ double* f1() const { return b + 12 * np; }
    __device__ double* fw() const { return b + 13 * np; }
    __device__ double* sv() const { return b + 14 * np; }
    __device__ double* srv() const { return b + 15 * np; }
};

// nodes eliminated at CR level lev (j = s-1 + 2s*m < n) and kept (j = 2s-1 + 2s*m < n)
__host__ __device__ __forceinline__ constexpr int lvl_count(int n, int lev) {
    return n >= (1 << lev) ? ((n - (1 << lev)) >> (lev + 1)) + 1 : 0;
}
__host__ __device__ __forceinline__ constexpr int kept_count(int n, int lev) {
    return n >> (lev + 1);
}
// number of leading levels with more than 32 eliminated nodes (run CTA-wide)
__host__ __device__ __forceinline__ constexpr int cta_levels(int n) {
    int l = 0;
    while (l < ilog2(n) && lvl_count(n, l) > 32) ++l;
    return l;
}

template <bool RHS>
struct CrSolve {
    // phase 1 at level lev for eliminated index m: invert D_p, snapshot lower coupling
    static __device__ __forceinline__ void elim(const TriSm& S, int n, int lev, int m) {
        const int s = 1 << lev;
        const int p = s - 1 + 2 * s * m;
        const int P = PI(p);
        const double a = S.Da()[P], b = S.Db()[P], c = S.Dc()[P];
        const double idet = 1.0 / (a * c - b * b);
        S.Da()[P] = c * idet;
        S.Db()[P] = -b * idet;
        S.Dc()[P] = a * idet;
        if (p - s >= 0) {
            const int Q = PI(p - s);
            S.L0()[P] = S.E0()[Q]; S.L1()[P] = S.E1()[Q];
            S.L2()[P] = S.E2()[Q]; S.L3()[P] = S.E3()[Q];
        } else {
            S.L0()[P] = 0.0; S.L1()[P] = 0.0; S.L2()[P] = 0.0; S.L3()[P] = 0.0;
        }
    }
    // phase 2 at level lev for kept index m: Schur update of D_j, E_j, f_j
    static __device__ __forceinline__ void keep(const TriSm& S, int n, int lev, int m,
                                                const double* cinv, const double* cup,
                                                const double* clo) {
        const int s = 1 << lev;
        const int j = 2 * s - 1 + 2 * s * m;
        const int p = j - s, q = j + s;
        const int J = PI(j), P = PI(p);
        double da = S.Da()[J], db = S.Db()[J], dc = S.Dc()[J];
        double g0 = 0.0, g1 = 0.0, w = 0.0;
        if (RHS) {
            g0 = S.f0()[J]; g1 = S.f1()[J];
            w = S.fw()[J] - cup[p] * cinv[p] * S.fw()[P];
        }
        {   // lower neighbour p: coupling A = E_p (row p, col j)
            const double e0 = S.E0()[P], e1 = S.E1()[P], e2 = S.E2()[P], e3 = S.E3()[P];
            const double pa = S.Da()[P], pb = S.Db()[P], pc = S.Dc()[P];
            const double t00 = e0 * pa + e2 * pb, t01 = e0 * pb + e2 * pc;
            const double t10 = e1 * pa + e3 * pb, t11 = e1 * pb + e3 * pc;
            da -= t00 * e0 + t01 * e2;
            db -= t00 * e1 + t01 * e3;
            dc -= t10 * e1 + t11 * e3;
            if (RHS) {
                const double h0 = S.f0()[P], h1 = S.f1()[P];
                g0 -= t00 * h0 + t01 * h1;
                g1 -= t10 * h0 + t11 * h1;
            }
        }
        double n0 = 0.0, n1 = 0.0, n2 = 0.0, n3 = 0.0;
        if (q < n) {  // upper neighbour q: coupling A = E_j (row j, col q)
            const int Qi = PI(q);
            const double e0 = S.E0()[J], e1 = S.E1()[J], e2 = S.E2()[J], e3 = S.E3()[J];
            const double qa = S.Da()[Qi], qb = S.Db()[Qi], qc = S.Dc()[Qi];
            const double t00 = e0 * qa + e1 * qb, t01 = e0 * qb + e1 * qc;
            const double t10 = e2 * qa + e3 * qb, t11 = e2 * qb + e3 * qc;
            da -= t00 * e0 + t01 * e1;
            db -= t00 * e2 + t01 * e3;
            dc -= t10 * e2 + t11 * e3;
            if (RHS) {
                const double h0 = S.f0()[Qi], h1 = S.f1()[Qi];
                g0 -= t00 * h0 + t01 * h1;
                g1 -= t10 * h0 + t11 * h1;
                w -= clo[q] * cinv[q] * S.fw()[Qi];
            }
            if (q + s < n) {
                const double k0 = S.E0()[Qi], k1 = S.E1()[Qi], k2 = S.E2()[Qi], k3 = S.E3()[Qi];
                n0 = -(t00 * k0 + t01 * k2);
                n1 = -(t00 * k1 + t01 * k3);
                n2 = -(t10 * k0 + t11 * k2);
                n3 = -(t10 * k1 + t11 * k3);
            }
        }
        S.Da()[J] = da; S.Db()[J] = db; S.Dc()[J] = dc;
        S.E0()[J] = n0; S.E1()[J] = n1; S.E2()[J] = n2; S.E3()[J] = n3;
        if (RHS) { S.f0()[J] = g0; S.f1()[J] = g1; S.fw()[J] = w; }
    }
    static __device__ __forceinline__ void root(const TriSm& S, int n, const double* cinv) {
        const int r = (1 << ilog2(n)) - 1, R = PI(r);
        const double a = S.Da()[R], b = S.Db()[R], c = S.Dc()[R];
        const double idet = 1.0 / (a * c - b * b);
        S.Da()[R] = c * idet; S.Db()[R] = -b * idet; S.Dc()[R] = a * idet;
        if (RHS) {
            const double g0 = S.f0()[R], g1 = S.f1()[R];
            S.f0()[R] = (c * g0 - b * g1) * idet;
            S.f1()[R] = (a * g1 - b * g0) * idet;
            S.fw()[R] = cinv[r] * S.fw()[R];
        } else {
            S.E0()[R] = 0.0; S.E1()[R] = 0.0; S.E2()[R] = 0.0; S.E3()[R] = 0.0;
            S.L0()[R] = 0.0; S.L1()[R] = 0.0; S.L2()[R] = 0.0; S.L3()[R] = 0.0;
        }
    }
    // back substitution at level lev for eliminated index m
    static __device__ __forceinline__ void back(const TriSm& S, int n, int lev, int m,
                                                const double* cinv, const double* cup,
                                                const double* clo) {
        const int s = 1 << lev;
        const int p = s - 1 + 2 * s * m;
        const int P = PI(p);
        double g0 = S.f0()[P], g1 = S.f1()[P], w = S.fw()[P];
        if (p - s >= 0) {
            const int Q = PI(p - s);
            const double xa = S.f0()[Q], xb = S.f1()[Q];
            g0 -= S.L0()[P] * xa + S.L2()[P] * xb;
            g1 -= S.L1()[P] * xa + S.L3()[P] * xb;
            w -= clo[p] * S.fw()[Q];
        }
        if (p + s < n) {
            const int Q = PI(p + s);
            const double xa = S.f0()[Q], xb = S.f1()[Q];
            g0 -= S.E0()[P] * xa + S.E1()[P] * xb;
            g1 -= S.E2()[P] * xa + S.E3()[P] * xb;
            w -= cup[p] * S.fw()[Q];
        }
        const double pa = S.Da()[P], pb = S.Db()[P], pc = S.Dc()[P];
        S.f0()[P] = pa * g0 + pb * g1;
        S.f1()[P] = pb * g0 + pc * g1;
        S.fw()[P] = cinv[p] * w;
    }
};

// One CTA-wide cyclic-reduction level (factorisation + rhs) with a single
// barrier.  Kept node j = 2s-1+2sm eliminates both neighbours p = j-s and
// q = j+s itself (each pivot is inverted by the two kept nodes that border
// it), so no separate elimination phase is needed.  j records for its upper
// neighbour q the lower coupling L_q = E_j (before updating E_j) and, after
// the barrier (when nobody reads the raw pivot any more), the inverse P_q in
// q's D slot; kept node m = 0 does the same for p = s-1.  The scalar Q_z
// reduction of fw rides along with the precomputed coefficients cr.
template <int KPT>
__device__ __forceinline__ void cr_level(const TriSm& S, int n, int lev,
                                         const double* __restrict__ cr) {
    const double* cinv = cr;
    const double* cup = cr + n;
    const double* clo = cr + 2 * n;
    const int s = 1 << lev, tid = threadIdx.x, nth = blockDim.x;
    const int ck = kept_count(n, lev);
    double qa[KPT], qb[KPT], qc[KPT];
    int qi[KPT];
    double p0a = 0.0, p0b = 0.0, p0c = 0.0;
    int p0i = -1;
#pragma unroll
    for (int t = 0; t < KPT; ++t) {
        qi[t] = -1;
        qa[t] = qb[t] = qc[t] = 0.0;
        const int m = tid + t * nth;
        if (m < ck) {
            const int j = 2 * s - 1 + 2 * s * m, p = j - s, q = j + s;
            const int J = PI(j), P = PI(p);
            double pa, pb, pc;
            {
                const double a = S.Da()[P], b = S.Db()[P], c = S.Dc()[P];
                const double id = 1.0 / (a * c - b * b);
                pa = c * id; pb = -b * id; pc = a * id;
            }
            if (m == 0) {
                p0a = pa; p0b = pb; p0c = pc; p0i = P;
                S.L0()[P] = 0.0; S.L1()[P] = 0.0; S.L2()[P] = 0.0; S.L3()[P] = 0.0;
            }
            double da = S.Da()[J], db = S.Db()[J], dc = S.Dc()[J];
            double g0 = S.f0()[J], g1 = S.f1()[J];
            double w = S.fw()[J] - cup[p] * cinv[p] * S.fw()[P];
            {   // lower neighbour p: coupling E_p (row p, col j)
                const double e0 = S.E0()[P], e1 = S.E1()[P], e2 = S.E2()[P], e3 = S.E3()[P];
                const double t00 = e0 * pa + e2 * pb, t01 = e0 * pb + e2 * pc;
                const double t10 = e1 * pa + e3 * pb, t11 = e1 * pb + e3 * pc;
                da -= t00 * e0 + t01 * e2;
                db -= t00 * e1 + t01 * e3;
                dc -= t10 * e1 + t11 * e3;
                const double h0 = S.f0()[P], h1 = S.f1()[P];
                g0 -= t00 * h0 + t01 * h1;
                g1 -= t10 * h0 + t11 * h1;
            }
            double n0 = 0.0, n1 = 0.0, n2 = 0.0, n3 = 0.0;
            if (q < n) {   // upper neighbour q: coupling E_j (row j, col q)
                const int Qi = PI(q);
                double xa, xb, xc;
                {
                    const double a = S.Da()[Qi], b = S.Db()[Qi], c = S.Dc()[Qi];
                    const double id = 1.0 / (a * c - b * b);
                    xa = c * id; xb = -b * id; xc = a * id;
                }
                const double e0 = S.E0()[J], e1 = S.E1()[J], e2 = S.E2()[J], e3 = S.E3()[J];
                S.L0()[Qi] = e0; S.L1()[Qi] = e1; S.L2()[Qi] = e2; S.L3()[Qi] = e3;
                const double t00 = e0 * xa + e1 * xb, t01 = e0 * xb + e1 * xc;
                const double t10 = e2 * xa + e3 * xb, t11 = e2 * xb + e3 * xc;
                da -= t00 * e0 + t01 * e1;
                db -= t00 * e2 + t01 * e3;
                dc -= t10 * e2 + t11 * e3;
                const double h0 = S.f0()[Qi], h1 = S.f1()[Qi];
                g0 -= t00 * h0 + t01 * h1;
                g1 -= t10 * h0 + t11 * h1;
                w -= clo[q] * cinv[q] * S.fw()[Qi];
                if (q + s < n) {
                    const double k0 = S.E0()[Qi], k1 = S.E1()[Qi], k2 = S.E2()[Qi], k3 = S.E3()[Qi];
                    n0 = -(t00 * k0 + t01 * k2);
                    n1 = -(t00 * k1 + t01 * k3);
                    n2 = -(t10 * k0 + t11 * k2);
                    n3 = -(t10 * k1 + t11 * k3);
                }
                qa[t] = xa; qb[t] = xb; qc[t] = xc; qi[t] = Qi;
            }
            S.Da()[J] = da; S.Db()[J] = db; S.Dc()[J] = dc;
            S.E0()[J] = n0; S.E1()[J] = n1; S.E2()[J] = n2; S.E3()[J] = n3;
            S.f0()[J] = g0; S.f1()[J] = g1; S.fw()[J] = w;
        }
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < KPT; ++t) {
        if (qi[t] >= 0) { S.Da()[qi[t]] = qa[t]; S.Db()[qi[t]] = qb[t]; S.Dc()[qi[t]] = qc[t]; }
    }
    if (p0i >= 0) { S.Da()[p0i] = p0a; S.Db()[p0i] = p0b; S.Dc()[p0i] = p0c; }
}

// The A <= 32 nodes left at the cut level, solved by parallel cyclic
// reduction in warp 0 with one node per lane (registers + shuffles, no
// back-substitution): each step eliminates the couplings at distance s with
// the neighbours' inverted pivots; the system stays symmetric, so the lower
// neighbour's upper coupling is this lane's lower coupling transposed.
__device__ __forceinline__ void pcr_tail(const TriSm& S, int c, int A) {
    const unsigned F = 0xffffffffu;
    const int m = threadIdx.x & 31;
    const bool act = m < A;
    const int J = act ? PI(((m + 1) << c) - 1) : 0;
    double da = 1.0, db = 0.0, dc = 1.0, u0 = 0.0, u1 = 0.0, u2 = 0.0, u3 = 0.0, f0 = 0.0, f1 = 0.0;
    if (act) {
        da = S.Da()[J]; db = S.Db()[J]; dc = S.Dc()[J];
        u0 = S.E0()[J]; u1 = S.E1()[J]; u2 = S.E2()[J]; u3 = S.E3()[J];
        f0 = S.f0()[J]; f1 = S.f1()[J];
    }
    // lower coupling (row m, col m-1) = E_{m-1}^T
    double l0 = __shfl_up_sync(F, u0, 1), l1 = __shfl_up_sync(F, u2, 1);
    double l2 = __shfl_up_sync(F, u1, 1), l3 = __shfl_up_sync(F, u3, 1);
    if (m == 0) { l0 = 0.0; l1 = 0.0; l2 = 0.0; l3 = 0.0; }
    for (int s = 1; s < A; s <<= 1) {
        const double id = 1.0 / (da * dc - db * db);
        const double ia = dc * id, ib = -db * id, ic = da * id;
        const double La = __shfl_up_sync(F, ia, s), Lb = __shfl_up_sync(F, ib, s),
                     Lc = __shfl_up_sync(F, ic, s);
        const double Ll0 = __shfl_up_sync(F, l0, s), Ll1 = __shfl_up_sync(F, l1, s),
                     Ll2 = __shfl_up_sync(F, l2, s), Ll3 = __shfl_up_sync(F, l3, s);
        const double Lf0 = __shfl_up_sync(F, f0, s), Lf1 = __shfl_up_sync(F, f1, s);
        const double Ua = __shfl_down_sync(F, ia, s), Ub = __shfl_down_sync(F, ib, s),
                     Uc = __shfl_down_sync(F, ic, s);
        const double Uu0 = __shfl_down_sync(F, u0, s), Uu1 = __shfl_down_sync(F, u1, s),
                     Uu2 = __shfl_down_sync(F, u2, s), Uu3 = __shfl_down_sync(F, u3, s);
        const double Uf0 = __shfl_down_sync(F, f0, s), Uf1 = __shfl_down_sync(F, f1, s);
        double a00 = 0.0, a01 = 0.0, a10 = 0.0, a11 = 0.0;
        double b00 = 0.0, b01 = 0.0, b10 = 0.0, b11 = 0.0;
        if (m >= s) {          // alpha = -Lo P_{m-s}
            a00 = -(l0 * La + l1 * Lb); a01 = -(l0 * Lb + l1 * Lc);
            a10 = -(l2 * La + l3 * Lb); a11 = -(l2 * Lb + l3 * Lc);
        }
        if (m + s < A) {       // beta = -Up P_{m+s}
            b00 = -(u0 * Ua + u1 * Ub); b01 = -(u0 * Ub + u1 * Uc);
            b10 = -(u2 * Ua + u3 * Ub); b11 = -(u2 * Ub + u3 * Uc);
        }
        da += a00 * l0 + a01 * l1 + b00 * u0 + b01 * u1;
        db += a00 * l2 + a01 * l3 + b00 * u2 + b01 * u3;
        dc += a10 * l2 + a11 * l3 + b10 * u2 + b11 * u3;
        f0 += a00 * Lf0 + a01 * Lf1 + b00 * Uf0 + b01 * Uf1;
        f1 += a10 * Lf0 + a11 * Lf1 + b10 * Uf0 + b11 * Uf1;
        l0 = a00 * Ll0 + a01 * Ll2; l1 = a00 * Ll1 + a01 * Ll3;
        l2 = a10 * Ll0 + a11 * Ll2; l3 = a10 * Ll1 + a11 * Ll3;
        u0 = b00 * Uu0 + b01 * Uu2; u1 = b00 * Uu1 + b01 * Uu3;
        u2 = b10 * Uu0 + b11 * Uu2; u3 = b10 * Uu1 + b11 * Uu3;
    }
    const double id = 1.0 / (da * dc - db * db);
    if (act) {
        S.f0()[J] = (dc * f0 - db * f1) * id;
        S.f1()[J] = (da * f1 - db * f0) * id;
    }
}

// Scalar Q_z system reduced to the cut: w_a = (Q_z^{-1})_aa fw_a (qzw
// transposed), one warp.
__device__ __forceinline__ void scal_cut(const TriSm& S, int c, int A,
                                         const double* __restrict__ qzw) {
    const int a = threadIdx.x & 31;
    double x = 0.0;
    if (a < A) {
        for (int m = 0; m < A; ++m) x = fma(qzw[m * A + a], S.fw()[PI(((m + 1) << c) - 1)], x);
    }
    __syncwarp();
    if (a < A) S.fw()[PI(((a + 1) << c) - 1)] = x;
}

// Block cyclic reduction of the symmetric quasi-definite 2x2-block tridiagonal
// system held in S (D sym (a,b,c), E upper coupling, f rhs), jointly with the
// scalar reduction of Qz w = fw (coefficients cr; reduced inverse qzw at the
// cut).  Levels below the cut run CTA-wide with one barrier each; the <= 32
// nodes at the cut by parallel cyclic reduction in warp 0 while warp 1 (or
// warp 0 afterwards) applies the scalar reduced inverse; then the CTA-wide
// back-substitution.  Solutions overwrite f0/f1/fw.
template <int KPT>
__device__ __forceinline__ void cr_solve(int n, const TriSm& S, const double* __restrict__ cr,
                                         const double* __restrict__ qzw) {
    using K = CrSolve<true>;
    const int tid = threadIdx.x, nth = blockDim.x;
    const double* cinv = cr;
    const double* cup = cr + n;
    const double* clo = cr + 2 * n;
    const int c = cut_level(n), A = cut_nodes(n);
#pragma unroll
    for (int lev = 0; lev < kMaxLev; ++lev) {
        if (lev >= c) break;
        cr_level<KPT>(S, n, lev, cr);
    }
    __syncthreads();
    if (tid < 32) {
        pcr_tail(S, c, A);
        if (nth <= 32) scal_cut(S, c, A, qzw);
    } else if (tid < 64) {
        scal_cut(S, c, A, qzw);
    }
    __syncthreads();
#pragma unroll
    for (int lev = kMaxLev - 1; lev >= 0; --lev) {
        if (lev >= c) continue;
        const int ce = lvl_count(n, lev);
        for (int m = tid; m < ce; m += nth) K::back(S, n, lev, m, cinv, cup, clo);
        __syncthreads();
    }
}

// Load D/E of the (u,lam) system of interval i into shared memory.
__device__ __forceinline__ void tri_init_de(const TView& V, int n, int i, const TriSm& S) {
    const Lay& L = V.lay;
    const double k2 = V.kappa * V.kappa;
    const double* Qu = (i == L.N - 1) ? V.Ql : V.Qm;
    const double* K = V.Ki(i, n);
    const double* Qz = V.Qz;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        const int J = PI(j);
        S.Da()[J] = Qu[n + j];
        S.Db()[J] = K[n + j];
        S.Dc()[J] = -k2 * Qz[n + j];
        if (j < n - 1) {
            S.E0()[J] = Qu[2 * n + j];
            S.E1()[J] = K[j + 1];
            S.E2()[J] = K[2 * n + j];
            S.E3()[J] = -k2 * Qz[2 * n + j];
        } else {
            S.E0()[J] = 0.0; S.E1()[J] = 0.0; S.E2()[J] = 0.0; S.E3()[J] = 0.0;
        }
    }
}

// One block row: residual (or given rhs) -> exact local KKT solve -> update.
//   r = b - (D x + couplings(uprev, munext))   (x, uprev, munext may be null)
//   out = (xupd ? xupd : 0) + omega * D^{-1} r
// Pointers that may be written by the same kernel (serial substitution) are
// read through plain loads (no __restrict__/.nc).
template <int NT>
__device__ __forceinline__ void tri_block(const TView& V, int i, const double* b, const double* x,
                                          const double* uprev, const double* munext, double* out,
                                          double omega, const double* xupd, double* sm) {
    const Lay& L = V.lay;
    const int n = dimn<NT>(V);
    const int tid = threadIdx.x, nth = blockDim.x;
    const bool has_vm = i >= 1, has_uzl = i < L.N;
    const TriSm S(sm, n);
    const double kap = V.kappa;
    const double* Qv = (i == L.N) ? V.Ql : V.Qm;
    const double* Qu = (i == L.N - 1) ? V.Ql : V.Qm;
    const double* Qz = V.Qz;
    const double* K = has_uzl ? V.Ki(i, n) : nullptr;
    const double* C = (has_uzl && has_vm) ? V.Ci(i, n) : nullptr;
    const int64_t bs = V.sl.base;
    const int64_t ov = L.off_v(i) - bs, ou = L.off_u(i) - bs, oz = L.off_z(i) - bs,
                  om = L.off_mu(i) - bs, ol = L.off_l(i) - bs;

    for (int j = tid; j < n; j += nth) {
        const int J = PI(j);
        double rv = 0.0, ru = 0.0, rz = 0.0, rm = 0.0, rl = 0.0;
        if (b) {
            if (has_vm) { rv = b[ov + j]; rm = b[om + j]; }
            if (has_uzl) { ru = b[ou + j]; rz = b[oz + j]; rl = b[ol + j]; }
        }
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
        if (has_vm) { S.sv()[J] = -rm; S.srv()[J] = rv; }
        if (has_uzl) { S.f0()[J] = ru; S.f1()[J] = rl - kap * rz; S.fw()[J] = rz; }
    }
    __syncthreads();
    if (!has_uzl) {  // last block (v_N, mu_N): mu = Qv v - r_v
        for (int j = tid; j < n; j += nth) {
            const double dv = S.sv()[PI(j)];
            const double dm = tmv_s(Qv, n, S.sv(), j) - S.srv()[PI(j)];
            const double bv = xupd ? xupd[ov + j] : 0.0, bm = xupd ? xupd[om + j] : 0.0;
            out[ov + j] = bv + omega * dv;
            out[om + j] = bm + omega * dm;
        }
        __syncthreads();
        return;
    }
    if (C) {
        for (int j = tid; j < n; j += nth) S.f1()[PI(j)] -= tmv_s(C, n, S.sv(), j);
    }
    tri_init_de(V, n, i, S);
    __syncthreads();
    cr_solve<(NT > 0 ? (NT / 2 + 127) / 128 : 4)>(n, S, V.cr, V.qzw);
    for (int j = tid; j < n; j += nth) {
        const int J = PI(j);
        const double du = S.f0()[J], dl = S.f1()[J];
        const double dz = S.fw()[J] - kap * dl;
        out[ou + j] = (xupd ? xupd[ou + j] : 0.0) + omega * du;
        out[oz + j] = (xupd ? xupd[oz + j] : 0.0) + omega * dz;
        out[ol + j] = (xupd ? xupd[ol + j] : 0.0) + omega * dl;
        if (has_vm) {
            const double dv = S.sv()[J];
            double dm = tmv_s(Qv, n, S.sv(), j) - S.srv()[J];
            if (C) dm += tmtv_s(C, n, S.f1(), j);
            out[ov + j] = (xupd ? xupd[ov + j] : 0.0) + omega * dv;
            out[om + j] = (xupd ? xupd[om + j] : 0.0) + omega * dm;
        }
    }
    __syncthreads();
}

// Parallel over block rows: jacobi (x may be null) or plain D^{-1} b.
template <int NT>
__global__ void __launch_bounds__(256, 3) tri_rows(TView V, const double* __restrict__ b,
                                                   const double* __restrict__ x,
                                                   double* __restrict__ y, double omega) {
    extern __shared__ __align__(16) double sm[];
    const Lay& L = V.lay;
    for (int i = V.sl.r0 + blockIdx.x; i < V.sl.r1; i += gridDim.x) {
        const double* uprev = x ? V.sl.uprev(L, x, i) : nullptr;
        const double* munext = x ? V.sl.munext(L, x, i) : nullptr;
        tri_block<NT>(V, i, b, x, uprev, munext, y, omega, x, sm);
    }
}

// Serial substitution over the time axis (smoothers.py:79-109), one CTA.
template <bool FORWARD, int NT>
__global__ void tri_subst(TView V, const double* __restrict__ r, double* d) {
    extern __shared__ __align__(16) double sm[];
    const Lay& L = V.lay;
    for (int k = 0; k <= L.N; ++k) {
        const int i = FORWARD ? k : L.N - k;
        const double* uprev = (FORWARD && i >= 1) ? d + L.off_u(i - 1) : nullptr;
        const double* munext = (!FORWARD && i < L.N) ? d + L.off_mu(i + 1) : nullptr;
        tri_block<NT>(V, i, r, nullptr, uprev, munext, d, 1.0, nullptr, sm);
    }
}

// ---------------------------------------------------------------------------
// Gauss-Seidel substitution as  parallel solve -> serial chain -> parallel solve.
// Forward (D-L)d = r:  d_i = D_i^{-1}(r_i - E_mu u_{i-1}), u_i = P_u d_i.  With
// a_i = D_i^{-1} r_i (parallel), the chain is  u_i = a_i^u + y_i, where y_i is
// the u-part of the (u,lam) solve with rhs (0, -C_i u_{i-1}).  Backward:
// mu_i = a_i^mu + C_i^T lam_i with lam_i from the rhs (-mu_{i+1}, 0).  The
// chain solves reuse per-interval cyclic-reduction factors precomputed once
// (fac record [14][n]: P(3) M1(4) M2(4) in CR level order, then C(3)),
// TMA bulk-staged in a double buffer so only the recurrences of the current
// interval sit on the serial critical path.
// ---------------------------------------------------------------------------
// Level order of the factor rows: node j = s-1 + 2s*m (s = 2^l) is eliminated
// at level l = ctz(j+1) with index m = (j+1) >> (l+1); level l occupies
// [lvl_off(l), lvl_off(l+1)).  Every CR level then reads a contiguous run.
__device__ __forceinline__ int lvl_pos(int n, int j) {
    const int lev = __ffs(j + 1) - 1;
    int off = 0;
    for (int l = 0; l < lev; ++l) off += lvl_count(n, l);
    return off + ((j + 1) >> (lev + 1));
}

// One CTA per interval i in [0, N): factor record of the (u,lam) system.
// Extra dynamic smem after the 16 node arrays: the 2A x 4A augmented matrix
// of the reduced system and a pivot column (Gauss-Jordan, no pivoting needed:
// the reduced system is symmetric quasi-definite).
// GW: the 16 node arrays live in global scratch (one slice per CTA) for n
// too large for shared memory.
template <int NT, bool GW>
__global__ void tri_factor_kernel(TView V, double* __restrict__ fac, double* gwork) {
    extern __shared__ __align__(16) double sm[];
    const Lay& L = V.lay;
    const int n = dimn<NT>(V);
    const int tid = threadIdx.x, nth = blockDim.x;
    const TriSm S(GW ? gwork + (size_t)blockIdx.x * kTriArrays * padded(n) : sm, n);
    const int c = cut_level(n), A = cut_nodes(n), M = 2 * A, M2 = 2 * M;
    double* G = GW ? sm : sm + kTriArrays * padded(n);   // [M][2M]
    double* fcol = G + M * M2;                           // [M]
    using K = CrSolve<false>;
    const double* cinv = V.cr;
    const int s1 = V.sl.r1 < L.N ? V.sl.r1 : L.N;         // stages of the slab
    for (int i = V.sl.r0 + blockIdx.x; i < s1; i += gridDim.x) {
        tri_init_de(V, n, i, S);
        __syncthreads();
        for (int lev = 0; lev < c; ++lev) {      // partial factorisation: levels < c
            const int ce = lvl_count(n, lev);
            for (int m = tid; m < ce; m += nth) K::elim(S, n, lev, m);
            __syncthreads();
            const int ck = kept_count(n, lev);
            for (int m = tid; m < ck; m += nth) K::keep(S, n, lev, m, cinv, cinv, cinv);
            __syncthreads();
        }
        // reduced system on the active nodes j_m = (m+1) 2^c - 1
        for (int e = tid; e < M * M2; e += nth) G[e] = 0.0;
        __syncthreads();
        for (int m = tid; m < A; m += nth) {
            const int J = PI(((m + 1) << c) - 1);
            const int r = 2 * m;
            G[r * M2 + r] = S.Da()[J];
            G[r * M2 + r + 1] = S.Db()[J];
            G[(r + 1) * M2 + r] = S.Db()[J];
            G[(r + 1) * M2 + r + 1] = S.Dc()[J];
            G[r * M2 + M + r] = 1.0;
            G[(r + 1) * M2 + M + r + 1] = 1.0;
            if (m + 1 < A) {
                const double e0 = S.E0()[J], e1 = S.E1()[J], e2 = S.E2()[J], e3 = S.E3()[J];
                G[r * M2 + r + 2] = e0; G[r * M2 + r + 3] = e1;
                G[(r + 1) * M2 + r + 2] = e2; G[(r + 1) * M2 + r + 3] = e3;
                G[(r + 2) * M2 + r] = e0; G[(r + 3) * M2 + r] = e1;
                G[(r + 2) * M2 + r + 1] = e2; G[(r + 3) * M2 + r + 1] = e3;
            }
        }
        __syncthreads();
        for (int k = 0; k < M; ++k) {            // Gauss-Jordan
            const double piv = G[k * M2 + k];
            for (int r = tid; r < M; r += nth) fcol[r] = (r == k) ? 0.0 : G[r * M2 + k] / piv;
            __syncthreads();
            for (int e = tid; e < M * M2; e += nth) {
                const int r = e / M2, col = e - r * M2;
                if (r != k) G[e] -= fcol[r] * G[k * M2 + col];
            }
            __syncthreads();
            for (int col = tid; col < M2; col += nth) G[k * M2 + col] /= piv;
            __syncthreads();
        }
        double* out = fac + (size_t)(i - V.sl.r0) * fac_record(n);
        const double* Cm = (i >= 1) ? V.Ci(i, n) : nullptr;
        for (int j = tid; j < n; j += nth) {
            const int lev = __ffs(j + 1) - 1;
            if (lev < c) {
                const int J = PI(j);
                const int o = lvl_pos(n, j);
                const double pa = S.Da()[J], pb = S.Db()[J], pc = S.Dc()[J];
                const double e0 = S.E0()[J], e1 = S.E1()[J], e2 = S.E2()[J], e3 = S.E3()[J];
                const double l0 = S.L0()[J], l1 = S.L1()[J], l2 = S.L2()[J], l3 = S.L3()[J];
                out[0 * n + o] = pa; out[1 * n + o] = pb; out[2 * n + o] = pc;
                out[3 * n + o] = e0 * pa + e2 * pb;  out[4 * n + o] = e0 * pb + e2 * pc;
                out[5 * n + o] = e1 * pa + e3 * pb;  out[6 * n + o] = e1 * pb + e3 * pc;
                out[7 * n + o] = l0 * pa + l1 * pb;  out[8 * n + o] = l0 * pb + l1 * pc;
                out[9 * n + o] = l2 * pa + l3 * pb;  out[10 * n + o] = l2 * pb + l3 * pc;
            }
            out[11 * n + j] = Cm ? Cm[j] : 0.0;
            out[12 * n + j] = Cm ? Cm[n + j] : 0.0;
            out[13 * n + j] = Cm ? Cm[2 * n + j] : 0.0;
        }
        double* W = out + kFacRows * n;           // W^T: W[col][row]
        for (int e = tid; e < M * M; e += nth) {
            const int r = e / M, col = e - r * M;
            W[col * M + r] = G[r * M2 + M + col];
        }
        __syncthreads();
    }
}

#ifdef TK_PROF
// phase timestamps of one chain step (debug builds only: -DTK_PROF)
__device__ long long g_tk_prof[16];
#define TKP(slot, cond)                                                  \
    do {                                                                 \
        if ((cond) && threadIdx.x == 0) g_tk_prof[slot] = clock64();     \
    } while (0)
#define TKA(slot, v)                                                     \
    do {                                                                 \
        if (threadIdx.x == 0 && blockIdx.x == 0) g_tk_prof[slot] += (v); \
    } while (0)
#define TKCLK() clock64()
// kernel-wide span of the grouped carry: [0] min CTA start, [1] max CTA end,
// [2] max start, [3] CTA 0 end - start (globaltimer ns)
__device__ unsigned long long g_tk_span[8] = {~0ull, 0ull, 0ull, 0ull, ~0ull, 0ull, 0ull, 0ull};
__device__ __forceinline__ unsigned long long tk_gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define TKSPAN_BEGIN(o)                                                  \
    unsigned long long tk_t0 = 0;                                        \
    if (threadIdx.x == 0) {                                              \
        tk_t0 = tk_gtime();                                              \
        atomicMin(&g_tk_span[(o) + 0], tk_t0);                           \
        atomicMax(&g_tk_span[(o) + 2], tk_t0);                           \
    }
#define TKSPAN_END(o)                                                    \
    if (threadIdx.x == 0) {                                              \
        const unsigned long long t1 = tk_gtime();                        \
        atomicMax(&g_tk_span[(o) + 1], t1);                              \
        if (blockIdx.x == 0) g_tk_span[(o) + 3] = t1 - tk_t0;            \
    }
#else
#define TKSPAN_BEGIN(o) \
    do {                \
    } while (0)
#define TKSPAN_END(o) \
    do {              \
    } while (0)
#define TKA(slot, v) \
    do {             \
    } while (0)
#define TKCLK() 0LL
#define TKP(slot, cond) \
    do {                \
    } while (0)
#endif

// forward rhs reduction of level lev for kept-node index m (level-ordered
// factors at off; record rows of length n at fb; f1 = f0 + np)
__device__ __forceinline__ void cr_rhs_down(const double* fb, int n, int np, int lev, int off,
                                            int m, double* f0) {
    double* f1 = f0 + np;
    const int s = 1 << lev;
    const int j = 2 * s - 1 + 2 * s * m;
    const int p = j - s, q = j + s;
    const int J = PI(j), P = PI(p), Pf = off + m;
    const double h0 = f0[P], h1 = f1[P];
    const double k0 = (q < n) ? f0[PI(q)] : 0.0, k1 = (q < n) ? f1[PI(q)] : 0.0;
    const int Qf = (q < n) ? Pf + 1 : Pf;
    const double t0 = fb[7 * n + Qf] * k0 + fb[8 * n + Qf] * k1;
    const double t1 = fb[9 * n + Qf] * k0 + fb[10 * n + Qf] * k1;
    f0[J] = fma(-fb[3 * n + Pf], h0, fma(-fb[4 * n + Pf], h1, f0[J])) - t0;
    f1[J] = fma(-fb[5 * n + Pf], h0, fma(-fb[6 * n + Pf], h1, f1[J])) - t1;
}

// back substitution of eliminated-node index m at level lev
__device__ __forceinline__ void cr_rhs_up(const double* fb, int n, int np, int lev, int off,
                                          int m, double* f0) {
    double* f1 = f0 + np;
    const int s = 1 << lev;
    const int p = s - 1 + 2 * s * m;
    const int P = PI(p), Pf = off + m;
    const double g0 = f0[P], g1 = f1[P];
    const double pa = fb[Pf], pb = fb[n + Pf], pc = fb[2 * n + Pf];
    double x0 = pa * g0 + pb * g1;
    double x1 = pb * g0 + pc * g1;
    if (p - s >= 0) {  // - M2_p^T x_{p-s}
        const int Q = PI(p - s);
        const double a = f0[Q], b = f1[Q];
        x0 -= fb[7 * n + Pf] * a + fb[9 * n + Pf] * b;
        x1 -= fb[8 * n + Pf] * a + fb[10 * n + Pf] * b;
    }
    if (p + s < n) {   // - M1_p^T x_{p+s}
        const int Q = PI(p + s);
        const double a = f0[Q], b = f1[Q];
        x0 -= fb[3 * n + Pf] * a + fb[5 * n + Pf] * b;
        x1 -= fb[4 * n + Pf] * a + fb[6 * n + Pf] * b;
    }
    f0[P] = x0;
    f1[P] = x1;
}

// scalar cyclic reduction of Qz w = fw with precomputed coefficients
// cr = [3][n] = (inv_d, e_up, e_lo) at each node's elimination level
__device__ __forceinline__ void scal_down(double* fw, const double* cr, int n, int lev, int m) {
    const int s = 1 << lev;
    const int j = 2 * s - 1 + 2 * s * m, p = j - s, q = j + s;
    double w = fw[PI(j)] - cr[n + p] * cr[p] * fw[PI(p)];
    if (q < n) w -= cr[2 * n + q] * cr[q] * fw[PI(q)];
    fw[PI(j)] = w;
}
__device__ __forceinline__ void scal_up(double* fw, const double* cr, int n, int lev, int m) {
    const int s = 1 << lev;
    const int p = s - 1 + 2 * s * m;
    double w = fw[PI(p)];
    if (p - s >= 0) w -= cr[2 * n + p] * fw[PI(p - s)];
    if (p + s < n) w -= cr[n + p] * fw[PI(p + s)];
    fw[PI(p)] = cr[p] * w;
}

// rhs-only solve with a factor record: cyclic-reduction levels below the cut
// (CTA-wide while more than 32 nodes are eliminated, then in warp 0), the
// reduced system by the dense inverse W, and the back-substitution.  With
// fw != null the scalar Qz system (coefficients cr, reduced inverse qzw at
// the cut) is solved alongside, sharing the barriers.
__device__ __forceinline__ void cr_rhs(int n, const double* fb, double* f0, double* part,
                                       bool prof = false, double* fw = nullptr,
                                       const double* cr = nullptr, const double* qzw = nullptr) {
    const int tid = threadIdx.x, nth = blockDim.x;
    const int np = padded(n);
    const int c = cut_level(n), A = cut_nodes(n), M = 2 * A;
    const int lw = cta_levels(n) < c ? cta_levels(n) : c;
    double* f1 = f0 + np;
    int off = 0;
#pragma unroll
    for (int lev = 0; lev < kMaxLev; ++lev) {   // CTA-wide levels
        if (lev >= lw) break;
        const int ck = kept_count(n, lev);
        for (int m = tid; m < ck; m += nth) {
            cr_rhs_down(fb, n, np, lev, off, m, f0);
            if (fw) scal_down(fw, cr, n, lev, m);
        }
        off += lvl_count(n, lev);
        __syncthreads();
    }
    TKP(2, prof);
    if (lw < c) {
        if (tid < 32) {                   // warp-level levels below the cut
            int o = off;
#pragma unroll
            for (int l = 0; l < kMaxLev; ++l) {
                if (l < lw) continue;
                if (l >= c) break;
                if (tid < kept_count(n, l)) {
                    cr_rhs_down(fb, n, np, l, o, tid, f0);
                    if (fw) scal_down(fw, cr, n, l, tid);
                }
                o += lvl_count(n, l);
                __syncwarp();
            }
        }
        __syncthreads();
    }
    if (fw) {   // scalar reduced system: w_a = (Qz^{-1})_aa fw_a (qzw transposed)
        double x = 0.0;
        if (tid < A) {
            for (int m = 0; m < A; ++m) x = fma(qzw[m * A + tid], fw[PI(((m + 1) << c) - 1)], x);
        }
        __syncthreads();
        if (tid < A) fw[PI(((tid + 1) << c) - 1)] = x;
    }
    // dense solve of the reduced system: x = W g on the A active nodes.  Row r
    // is split over G = nth / M thread groups (column chunks); partial sums
    // meet in the shared scratch `part` ([blockDim.x] doubles).
    {
        const double* Wt = fb + kFacRows * n;
        if (nth >= M) {
            const int G = nth / M;
            const int r = tid % M, grp = tid / M;
            double acc0 = 0.0, acc1 = 0.0;
            if (grp < G) {
                const int per = (A + G - 1) / G;   // columns come in (u, lam) pairs per node
                const int m0 = grp * per, m1 = min(A, m0 + per);
                for (int m = m0; m < m1; ++m) {
                    const int J = PI(((m + 1) << c) - 1);
                    acc0 = fma(Wt[(2 * m) * M + r], f0[J], acc0);
                    acc1 = fma(Wt[(2 * m + 1) * M + r], f1[J], acc1);
                }
                part[tid] = acc0 + acc1;
            }
            __syncthreads();
            if (tid < M) {
                double x = 0.0;
                for (int g = 0; g < G; ++g) x += part[g * M + tid];
                const int J = PI(((tid >> 1) + 1 << c) - 1);
                (tid & 1 ? f1 : f0)[J] = x;
            }
        } else {                           // fewer threads than rows: whole rows per thread
            for (int r = tid; r < M; r += nth) {
                double acc0 = 0.0, acc1 = 0.0;
                for (int m = 0; m < A; ++m) {
                    const int J = PI(((m + 1) << c) - 1);
                    acc0 = fma(Wt[(2 * m) * M + r], f0[J], acc0);
                    acc1 = fma(Wt[(2 * m + 1) * M + r], f1[J], acc1);
                }
                part[r] = acc0 + acc1;
            }
            __syncthreads();
            for (int r = tid; r < M; r += nth) {
                const int J = PI(((r >> 1) + 1 << c) - 1);
                (r & 1 ? f1 : f0)[J] = part[r];
            }
        }
        __syncthreads();
    }
    TKP(3, prof);
    if (lw < c) {
        if (tid < 32) {                   // warp-level back-substitution
            int o = off;
            for (int l = lw; l < c; ++l) o += lvl_count(n, l);
#pragma unroll
            for (int l = kMaxLev - 1; l >= 0; --l) {
                if (l >= c || l < lw) continue;
                const int ce = lvl_count(n, l);
                o -= ce;
                if (tid < ce) {
                    cr_rhs_up(fb, n, np, l, o, tid, f0);
                    if (fw) scal_up(fw, cr, n, l, tid);
                }
                __syncwarp();
            }
        }
        __syncthreads();
    }
    TKP(4, prof);
#pragma unroll
    for (int lev = kMaxLev - 1; lev >= 0; --lev) {  // CTA-wide back-substitution
        if (lev >= lw) continue;
        const int ce = lvl_count(n, lev);
        off -= ce;
        for (int m = tid; m < ce; m += nth) {
            cr_rhs_up(fb, n, np, lev, off, m, f0);
            if (fw) scal_up(fw, cr, n, lev, m);
        }
        __syncthreads();
    }
    TKP(5, prof);
}

// --- TMA bulk copies + mbarrier (sm_90+; SASS UBLKCP / SYNCS) -------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_g2s(void* dst, const void* src, unsigned bytes,
                                        uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// L2 bulk prefetch of [p, p + bytes) (bytes a multiple of 16, p 16-byte aligned)
__device__ __forceinline__ void l2_prefetch_bulk(const void* p, unsigned bytes) {
    if (bytes == 0) return;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred P1;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        " @!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity)
        : "memory");
}

// Coupling chain over the steps of one time chunk (one CTA per chunk).
// FWD: chain[i] = u_i, BWD: chain[i] = mu_i; step k handles interval
// FWD ? 1+k : N-1-k.  The chunks partition the intervals 1..N-1 into runs of
// Lc (the same runs in both directions, so the backward chunk propagator is
// the transpose of the forward one); chunk c = cbase + blockIdx.x.  The chunk
// holding step 0 starts from the seed a_{i0} (and writes chain[i0]); the
// others start from starts[c*n] (zero when starts is null).  ends != null:
// the chunk's last value goes to ends[c*n].  HOM: homogeneous chain (a = 0)
// from the unit vector e_y (y = blockIdx.y); its end value is column y of the
// chunk propagator Pi_c, written to ends[(c*n + y)*n] (row y of Pi_c^T).
// `a` = D^{-1} r from pass 1.  STAGED: the next interval's record and
// a-segment are TMA bulk-copied into the other half of a double buffer while
// the current interval is solved.  The output of step k and the right-hand
// side of step k+1 are formed in one pass (two ping-pong rhs buffers).
template <bool FWD, bool STAGED, bool HOM, int NT>
__global__ void tri_chain_kernel(TView V, const double* __restrict__ a,
                                 const double* __restrict__ fac, double* __restrict__ chain,
                                 int Lc, int cbase, const double* __restrict__ starts,
                                 double* __restrict__ ends, int span = 1) {
    extern __shared__ __align__(16) double sm[];
    __shared__ __align__(8) uint64_t bars[2];
    const Lay& L = V.lay;
    const int n = dimn<NT>(V), N = L.N, np = padded(n);
    const int tid = threadIdx.x, nth = blockDim.x;
    const int rec = fac_record(n);
    const int brec = rec + n;
    double* buf0 = sm;
    double* buf1 = STAGED ? sm + brec : sm;
    double* fbase = STAGED ? sm + 2 * brec : sm;
    double* fr[2] = {fbase, fbase + 2 * np};
    const int K = N - 1;  // chain steps after the seed
    const int c = cbase + blockIdx.x * span;
    int hi0 = min(K, c * Lc + span * Lc);
    if (span > 1) hi0 = min(hi0, ((K + Lc - 1) / Lc - 1) * Lc);   // groups stop before the last chunk
    const int lo = c * Lc, hi = hi0;
    const int k0 = FWD ? lo : K - hi, k1 = FWD ? hi : K - lo;
    const bool seed = !HOM && k0 == 0;
    auto blk = [&](int k) { return FWD ? 1 + k : N - 1 - k; };
    auto aseg = [&](int i) { return a + (FWD ? L.off_u(i) : L.off_mu(i)); };
    auto record = [&](int k) -> const double* {
        return STAGED ? (((k - k0) & 1) ? buf1 : buf0) : fac + (size_t)blk(k) * rec;
    };
    auto aval = [&](int k) -> const double* { return STAGED ? record(k) + rec : aseg(blk(k)); };
    const int i0 = FWD ? 0 : N;
    const double* s0 = seed ? aseg(i0) : (HOM ? nullptr : (starts ? starts + (size_t)c * n : nullptr));
    const int ey = blockIdx.y;
    auto startv = [&](int j) -> double {
        if (HOM) return j == ey ? 1.0 : 0.0;
        return s0 ? s0[j] : 0.0;
    };
    if (seed) {
        for (int j = tid; j < n; j += nth) chain[(size_t)i0 * n + j] = s0[j];
    }
    if (k0 >= k1) return;
    const int pt = nth - 1;        // the thread issuing the TMA prefetches
    if (STAGED && tid == pt) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    auto prefetch = [&](int k) {
        const int t = k - k0;
        double* b = (t & 1) ? buf1 : buf0;
        uint64_t* bar = &bars[t & 1];
        const int i = blk(k);
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        mbar_expect_tx(bar, (unsigned)((HOM ? rec : brec) * sizeof(double)));
        tma_g2s(b, fac + (size_t)i * rec, (unsigned)(rec * sizeof(double)), bar);
        if (!HOM) tma_g2s(b + rec, aseg(i), (unsigned)(n * sizeof(double)), bar);
    };
    if (STAGED && tid == pt) prefetch(k0);
    if (STAGED) mbar_wait(&bars[0], 0u);
    {   // right-hand side of the first step from the start vector
        const double* fb = record(k0);
        const double *Cs = fb + 11 * n, *Cd = fb + 12 * n, *Cp = fb + 13 * n;
        double* f0 = fr[0];
        double* f1 = f0 + np;
        for (int j = tid; j < n; j += nth) {
            const int J = PI(j);
            if (FWD) {
                double cv = Cd[j] * startv(j);
                if (j > 0) cv += Cs[j] * startv(j - 1);
                if (j < n - 1) cv += Cp[j] * startv(j + 1);
                f0[J] = 0.0;
                f1[J] = -cv;
            } else {
                f0[J] = -startv(j);
                f1[J] = 0.0;
            }
        }
    }
    __syncthreads();
    double* eout = ends ? (HOM ? ends + ((size_t)(c / span) * n + ey) * n : ends + (size_t)c * n) : nullptr;
    for (int k = k0; k < k1; ++k) {
        const int t = k - k0;
        const int i = blk(k);
        const bool prof = !HOM && (k == K / 2);
        TKP(0, prof);
        if (STAGED && tid == pt && k + 1 < k1) prefetch(k + 1);
        const double* fb = record(k);
        const double* ai = HOM ? nullptr : aval(k);
        double* f0 = fr[t & 1];
        double* f1 = f0 + np;
        TKP(1, prof);
        cr_rhs(n, fb, f0, fbase + 4 * np, prof);
        const bool more = k + 1 < k1;
        if (STAGED && more) mbar_wait(&bars[(t + 1) & 1], (unsigned)(((t + 1) >> 1) & 1));
        const double* fbn = more ? record(k + 1) : fb;
        double* g0 = fr[(t + 1) & 1];
        double* g1 = g0 + np;
        const double *Cs = fb + 11 * n, *Cd = fb + 12 * n, *Cp = fb + 13 * n;
        const double *Ns = fbn + 11 * n, *Nd = fbn + 12 * n, *Np = fbn + 13 * n;
        for (int j = tid; j < n; j += nth) {
            const int J = PI(j);
            if (FWD) {   // u_i = a + u-part; next rhs (0, -C_{i+1} u_i)
                const double val = HOM ? f0[J] : ai[j] + f0[J];
                if (!HOM) chain[(size_t)i * n + j] = val;
                if (more) {
                    double cv = Nd[j] * val;
                    if (j > 0) cv += Ns[j] * (HOM ? f0[PI(j - 1)] : ai[j - 1] + f0[PI(j - 1)]);
                    if (j < n - 1) cv += Np[j] * (HOM ? f0[PI(j + 1)] : ai[j + 1] + f0[PI(j + 1)]);
                    g0[J] = 0.0;
                    g1[J] = -cv;
                } else if (eout) {
                    eout[j] = val;
                }
            } else {     // mu_i = a + C^T lam; next rhs (-mu_i, 0)
                double ct = Cd[j] * f1[J];
                if (j > 0) ct += Cp[j - 1] * f1[PI(j - 1)];
                if (j < n - 1) ct += Cs[j + 1] * f1[PI(j + 1)];
                const double val = HOM ? ct : ai[j] + ct;
                if (!HOM) chain[(size_t)i * n + j] = val;
                if (more) {
                    g0[J] = -val;
                    g1[J] = 0.0;
                } else if (eout) {
                    eout[j] = val;
                }
            }
        }
        (void)Ns; (void)Nd; (void)Np;
        __syncthreads();
        TKP(6, prof);
    }
}

// shared::cluster address of the same shared-memory location in CTA `rank`
__device__ __forceinline__ unsigned mapa_u32(unsigned a, unsigned rank) {
    unsigned d;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(d) : "r"(a), "r"(rank));
    return d;
}
// 8-byte store into a peer CTA's shared memory that completes 8 transaction
// bytes on the peer's mbarrier
__device__ __forceinline__ void st_async_f64(unsigned raddr, double v, unsigned rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];\n"
                 ::"r"(raddr), "l"(__double_as_longlong(v)), "r"(rbar)
                 : "memory");
}

// Register-row variant of the carry matvec (staged == 2: n % 64 == 0, n <= 512
// and exactly one row per warp): the lane's 16 entries of its row of the NEXT
// propagator are loaded into registers right after the current ones have been
// consumed, so they fly while the new U is pushed and awaited; shared memory
// then carries only U (the TMA-staged row block doubled its traffic: 256 KB
// per step and CTA at 128 B/clk was the step's largest part).  Same order of
// the products and sums as the staged loop.
static constexpr int kCarryNI = 16;
#ifndef TK_CARRY_AHEAD
#define TK_CARRY_AHEAD 2
#endif
static constexpr int kCarryAhead = TK_CARRY_AHEAD;   // row blocks prefetched into L2 ahead of the step
__device__ __forceinline__ void carry_loadrow(const double* __restrict__ row, int n, int lane,
                                              double (&m)[kCarryNI]) {
#pragma unroll
    for (int i = 0; i < kCarryNI; ++i) m[i] = (32 * i < n) ? __ldcg(row + lane + 32 * i) : 0.0;
}
__device__ __forceinline__ double carry_dotrow(const double (&m)[kCarryNI],
                                               const double* __restrict__ cur, int n, int lane) {
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int i = 0; i < kCarryNI; i += 2)
        if (32 * i < n) {
            a0 = fma(m[i], cur[lane + 32 * i], a0);
            a1 = fma(m[i + 1], cur[lane + 32 * i + 32], a1);
        }
    return a0 + a1;
}

// Serial carry over the chunk ends (one thread-block cluster):
//   U = ends[first];  for each next chunk c in chain order:
//     starts[c] = U;  U = ends[c] + M_c U
// with M_c = Pi_c (forward) or Pi_c^T (backward), row-major n x n.  Each CTA
// owns a block of rows of the matvec and pushes every new entry of U into
// all CTAs' shared copies with st.async; each copy (ping-pong by step) has
// an mbarrier expecting the n*8 bytes of one U, so the only synchronisation
// per chunk is that transaction count (no cluster-wide barrier).  staged:
// the CTA's row block of the next M_c is TMA bulk-copied into shared memory
// as soon as the current one has been consumed.
template <bool FWD, bool RG = false>
__global__ void __launch_bounds__(1024, 1)
    tri_chain_carry(int n, int nc, const double* __restrict__ M, const double* __restrict__ ends,
                    double* __restrict__ starts, int staged) {
    extern __shared__ __align__(16) double sm[];   // U ping-pong [2][n], row block
    __shared__ __align__(8) uint64_t tbar;          // TMA row block
    __shared__ __align__(8) uint64_t ubar[2];       // U copies
    cg::cluster_group cl = cg::this_cluster();
    const int CS = (int)cl.num_blocks();
    const int rank = (int)cl.block_rank();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    const int rpc = (n + CS - 1) / CS;
    const int r0 = min(n, rank * rpc), r1 = min(n, r0 + rpc);
    double* blk = sm + 2 * n;
    const unsigned bytes = (unsigned)((size_t)(r1 - r0) * n * sizeof(double));
    constexpr bool rg = RG;                      // register rows (one per warp)
    const bool stg = !RG && staged == 1 && bytes > 0;
    const unsigned ubytes = (unsigned)(n * sizeof(double));
    auto chunk_at = [&](int t) { return FWD ? t : nc - 1 - t; };
    double m[kCarryNI];
    auto rowp = [&](int t) { return M + (size_t)chunk_at(t) * n * n + (size_t)(r0 + warp) * n; };
    auto pf = [&](int t) {   // this CTA's row block of step t -> L2
        if (t < nc - 1) l2_prefetch_bulk(M + (size_t)chunk_at(t) * n * n + (size_t)r0 * n, bytes);
    };
    auto issue = [&](int t) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        mbar_expect_tx(&tbar, bytes);
        tma_g2s(blk, M + (size_t)chunk_at(t) * n * n + (size_t)r0 * n, bytes, &tbar);
        // the single staging buffer exposes this copy's latency every transition: pull the
        // next two row blocks into L2 now, so that their copies are L2 hits
        for (int a = 1; a <= 2; ++a)
            if (t + a < nc - 1)
                l2_prefetch_bulk(M + (size_t)chunk_at(t + a) * n * n + (size_t)r0 * n, bytes);
    };
    if (tid == 0) {
        mbar_init(&tbar, 1);
        mbar_init(&ubar[0], 1);
        mbar_init(&ubar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (stg && tid == 0 && nc > 2) issue(1);
    if (rg && nc > 2) {
        // the row blocks of the next kCarryAhead steps -> L2 (2 measured best: 4 and 8
        // ahead slow the forward substitution by 25-35 us)
        if (tid == 0)
            for (int a = 2; a < 2 + kCarryAhead; ++a) pf(a);
        carry_loadrow(rowp(1), n, lane, m);
    }
    const int first = FWD ? 0 : nc - 1;
    for (int j = tid; j < n; j += blockDim.x) sm[j] = ends[(size_t)first * n + j];
    cl.sync();   // every CTA's barriers are initialised before any st.async
    unsigned tphase = 0;
    for (int t = 1; t < nc; ++t) {
        const int c = chunk_at(t);
        long long c0 = TKCLK();
        if (t >= 2) mbar_wait(&ubar[(t - 1) & 1], (unsigned)(((t - 2) >> 1) & 1));
        long long c1 = TKCLK();
        TKA(8, c1 - c0);
        const double* cur = sm + ((t - 1) & 1) * n;
        for (int j = r0 + tid; j < r1; j += blockDim.x) starts[(size_t)c * n + j] = cur[j];
        if (t == nc - 1) break;
        if (tid == 0) mbar_expect_tx(&ubar[t & 1], ubytes);   // arm the copy of U_t
        c0 = TKCLK();
        if (stg) { mbar_wait(&tbar, tphase); tphase ^= 1u; }
        c1 = TKCLK();
        TKA(9, c1 - c0);
        const double* src = stg ? blk : M + (size_t)c * n * n + (size_t)r0 * n;
        const double* ec = ends + (size_t)c * n;
        const unsigned nxt = smem_u32(sm + (t & 1) * n);
        const unsigned bar = smem_u32(&ubar[t & 1]);
        if (rg) {
            const int r = r0 + warp;
            const double e = ec[r];
            double acc = carry_dotrow(m, cur, n, lane);
            if (t + 1 < nc - 1) carry_loadrow(rowp(t + 1), n, lane, m);
            if (tid == 0) pf(t + 1 + kCarryAhead);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            const double v = e + acc;
            for (int d = lane; d < CS; d += 32)
                st_async_f64(mapa_u32(nxt + 8u * r, d), v, mapa_u32(bar, d));
            TKA(10, TKCLK() - c1);
            __syncthreads();   // the warps stay within one step of each other
            continue;
        }
        for (int r = r0 + warp; r < r1; r += nw) {
            const double* row = src + (size_t)(r - r0) * n;
            const double e = ec[r];
            double a0 = 0.0, a1 = 0.0;
            int k = lane;
            for (; k + 32 < n; k += 64) {
                a0 = fma(row[k], cur[k], a0);
                a1 = fma(row[k + 32], cur[k + 32], a1);
            }
            if (k < n) a0 = fma(row[k], cur[k], a0);
            double acc = a0 + a1;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            const double v = e + acc;
            for (int d = lane; d < CS; d += 32)
                st_async_f64(mapa_u32(nxt + 8u * r, d), v, mapa_u32(bar, d));
        }
        TKA(10, TKCLK() - c1);
        if (stg) {
            __syncthreads();   // row block consumed: refill with the next chunk's
            if (tid == 0 && t + 1 < nc - 1) issue(t + 1);
        }
    }
    cl.sync();   // no CTA leaves while peers may still write into it
}

// Grouped carry (two-level scan of the chunk recurrence).  The transitions
// over chunks 1..nc-2 are split into groups of G consecutive chunks (group g:
// chunks [1+gG, min(nc-2, (g+1)G)]), one thread-block cluster per group.
//   mode 1 (phase A, all groups at once): run the group's transitions from
//     zero -- or, for the group first in chain order, from the exact seed
//     ends[first] (writing the exact starts) -- and store the group's end
//     value in GE[g];
//   phase B (tri_chain_carry over the groups with the group propagators Phi_g
//     and GE as the ends): exact group starts GS[g];
//   mode 2 (phase C, all groups but the first in chain order): re-run the
//     transitions from GS[g], writing the exact chunk starts.
// The group last in chain order also writes the start of the final chunk.
// Serial depth: 2G + nc/G matvecs instead of nc.
template <bool FWD, bool RG = false>
__global__ void __launch_bounds__(1024, 1)
    tri_chain_carry_seg(int n, int nc, int G, int mode, const double* __restrict__ M,
                        const double* __restrict__ ends, double* __restrict__ starts,
                        double* __restrict__ GE, const double* __restrict__ GS, int staged,
                        const double* __restrict__ Phi) {
    extern __shared__ __align__(16) double sm[];   // U ping-pong [2][n], row block
    __shared__ __align__(8) uint64_t tbar;
    __shared__ __align__(8) uint64_t ubar[2];
    TKSPAN_BEGIN(mode >= 2 ? 4 : 0);
    long long cp = TKCLK();
    cg::cluster_group cl = cg::this_cluster();
    const int CS = (int)cl.num_blocks();
    const int rank = (int)cl.block_rank();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    const int ng = (nc - 2 + G - 1) / G;
    const int q = blockIdx.x / CS;
    const int gi = (mode >= 2 && FWD) ? q + 1 : q;
    const bool first = FWD ? gi == 0 : gi == ng - 1;
    const bool last = FWD ? gi == ng - 1 : gi == 0;
    const int lo = 1 + gi * G, hi = min(nc - 2, (gi + 1) * G);
    const int L = hi - lo + 1;
    auto chunk_of = [&](int t) { return FWD ? lo + t : hi - t; };
    const int rpc = (n + CS - 1) / CS;
    const int r0 = min(n, rank * rpc), r1 = min(n, r0 + rpc);
    double* blk = sm + 2 * n;
    const unsigned bytes = (unsigned)((size_t)(r1 - r0) * n * sizeof(double));
    constexpr bool rg = RG;                      // register rows (one per warp)
    const bool stg = !RG && staged == 1 && bytes > 0;
    const unsigned ubytes = (unsigned)(n * sizeof(double));
    // mode 3: P prelude steps of the group-start recurrence (phase B's
    // GS[g'] = GE[g] + Phi_g GS[g], from the exact GE of the group first in
    // chain order) run by every cluster up to its own group, then the L
    // transitions of mode 2 -- same mat-vecs in the same order as phase B
    const int P = mode == 3 ? (FWD ? gi - 1 : ng - 2 - gi) : 0;
    const int LT = P + L;
    auto mat_of = [&](int t) -> const double* {   // n x n propagator of step t
        if (t < P) return Phi + (size_t)(FWD ? 1 + t : ng - 2 - t) * n * n;
        return M + (size_t)chunk_of(t - P) * n * n;
    };
    auto end_of = [&](int t) -> const double* {
        if (t < P) return GE + (size_t)(FWD ? 1 + t : ng - 2 - t) * n;
        return ends + (size_t)chunk_of(t - P) * n;
    };
    double m[kCarryNI];
    auto rowp = [&](int t) { return mat_of(t) + (size_t)(r0 + warp) * n; };
    auto pf = [&](int t) {   // this CTA's row block of step t -> L2
        if (t < LT) l2_prefetch_bulk(mat_of(t) + (size_t)r0 * n, bytes);
    };
    auto issue = [&](int t) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        mbar_expect_tx(&tbar, bytes);
        tma_g2s(blk, mat_of(t) + (size_t)r0 * n, bytes, &tbar);
        for (int a = 1; a <= 2; ++a)   // the next two row blocks -> L2 (see tri_chain_carry)
            if (t + a < LT) l2_prefetch_bulk(mat_of(t + a) + (size_t)r0 * n, bytes);
    };
    if (tid == 0) {
        mbar_init(&tbar, 1);
        mbar_init(&ubar[0], 1);
        mbar_init(&ubar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (stg && tid == 0 && LT > 0) issue(0);
    if (rg && LT > 0) {
        if (tid == 0)
            for (int a = 1; a < 1 + kCarryAhead; ++a) pf(a);
        carry_loadrow(rowp(0), n, lane, m);
    }
    const double* init = mode == 3 ? GE + (size_t)(FWD ? 0 : ng - 1) * n
                         : mode == 2 ? GS + (size_t)gi * n
                                     : (first ? ends + (size_t)(FWD ? 0 : nc - 1) * n : nullptr);
    for (int j = tid; j < n; j += blockDim.x) sm[j] = init ? init[j] : 0.0;
    cl.sync();   // every CTA's barriers are initialised before any st.async
    const bool wstart = mode >= 2 || first;
    unsigned tphase = 0;
    TKA(0, TKCLK() - cp);
    for (int t = 0; t < LT; ++t) {   // step t: U_{t+1} = E_c + M_c U_t
        const int c = chunk_of(t >= P ? t - P : 0);
        long long c0 = TKCLK();
        if (t >= 1) mbar_wait(&ubar[t & 1], (unsigned)(((t - 1) >> 1) & 1));
        long long c1 = TKCLK();
        TKA(12, c1 - c0);
        const double* cur = sm + (t & 1) * n;
        if (wstart && t >= P)
            for (int j = r0 + tid; j < r1; j += blockDim.x) starts[(size_t)c * n + j] = cur[j];
        if (tid == 0) mbar_expect_tx(&ubar[(t + 1) & 1], ubytes);   // arm the copy of U_{t+1}
        c0 = TKCLK();
        TKA(1, c0 - c1);
        if (stg) { mbar_wait(&tbar, tphase); tphase ^= 1u; }
        c1 = TKCLK();
        TKA(13, c1 - c0);
        const double* src = stg ? blk : mat_of(t) + (size_t)r0 * n;
        const double* ec = end_of(t);
        const unsigned nxt = smem_u32(sm + ((t + 1) & 1) * n);
        const unsigned bar = smem_u32(&ubar[(t + 1) & 1]);
        if (rg) {
            const int r = r0 + warp;
            const double e = ec[r];
            double acc = carry_dotrow(m, cur, n, lane);
            if (t + 1 < LT) carry_loadrow(rowp(t + 1), n, lane, m);
            if (tid == 0) pf(t + 1 + kCarryAhead);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            const double v = e + acc;
            for (int d = lane; d < CS; d += 32)
                st_async_f64(mapa_u32(nxt + 8u * r, d), v, mapa_u32(bar, d));
            c0 = TKCLK();
            TKA(14, c0 - c1);
            __syncthreads();   // the warps stay within one step of each other
            TKA(2, TKCLK() - c0);
            continue;
        }
        for (int r = r0 + warp; r < r1; r += nw) {
            const double* row = src + (size_t)(r - r0) * n;
            const double e = ec[r];
            double a0 = 0.0, a1 = 0.0;
            int k = lane;
            for (; k + 32 < n; k += 64) {
                a0 = fma(row[k], cur[k], a0);
                a1 = fma(row[k + 32], cur[k + 32], a1);
            }
            if (k < n) a0 = fma(row[k], cur[k], a0);
            double acc = a0 + a1;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            const double v = e + acc;
            for (int d = lane; d < CS; d += 32)
                st_async_f64(mapa_u32(nxt + 8u * r, d), v, mapa_u32(bar, d));
        }
        c0 = TKCLK();
        TKA(14, c0 - c1);
        if (stg) {
            __syncthreads();   // row block consumed: refill with the next transition's
            if (tid == 0 && t + 1 < LT) issue(t + 1);
        }
        TKA(2, TKCLK() - c0);
    }
    cp = TKCLK();
    if (LT > 0) mbar_wait(&ubar[LT & 1], (unsigned)(((LT - 1) >> 1) & 1));
    const double* fin = sm + (LT & 1) * n;
    if (mode == 1)
        for (int j = r0 + tid; j < r1; j += blockDim.x) GE[(size_t)gi * n + j] = fin[j];
    if (last && (mode >= 2 || first)) {
        const int cf = FWD ? nc - 1 : 0;
        for (int j = r0 + tid; j < r1; j += blockDim.x) starts[(size_t)cf * n + j] = fin[j];
    }
    cl.sync();   // no CTA leaves while peers may still write into it
    TKA(3, TKCLK() - cp);
    TKSPAN_END(mode >= 2 ? 4 : 0);
}

// Grid-wide variant of the carry (one CTA per SM, cooperative launch): CTA g
// owns rows [g R, g R + R) of every M_c.  Its row blocks are streamed by TMA
// into a ring of D shared-memory slots up to D chunks ahead, so the HBM
// traffic (n^2 doubles per chunk) runs at full-chip bandwidth off the serial
// path.  U_t goes through global memory (Ug, read with .cg loads) and one
// arrival counter (release/acquire) per chunk; the last CTA out resets the
// counters for the next launch.  D == 0: rows are loaded directly.
static constexpr int kCarryRing = 8;
template <bool FWD>
__global__ void __launch_bounds__(256, 1)
    tri_chain_carry_grid(int n, int nc, const double* __restrict__ M,
                         const double* __restrict__ ends, double* __restrict__ starts,
                         double* Ug, unsigned* cnt, int R, int D) {
    extern __shared__ __align__(16) double sm[];   // ring [D][R*n], then U [n]
    __shared__ __align__(8) uint64_t bars[kCarryRing];
    const int G = gridDim.x, g = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    const int r0 = min(n, g * R), r1 = min(n, r0 + R);
    const size_t slot = (size_t)R * n;
    double* Us = sm + (size_t)D * slot;
    const unsigned bytes = (unsigned)((size_t)(r1 - r0) * n * sizeof(double));
    const int T = nc - 2;   // chunks with a matvec: t = 1..T
    auto chunk_at = [&](int t) { return FWD ? t : nc - 1 - t; };
    auto issue = [&](int t) {   // row block of step t into slot (t-1) % D
        const int sl = (t - 1) % D;
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        mbar_expect_tx(&bars[sl], bytes);
        tma_g2s(sm + sl * slot, M + (size_t)chunk_at(t) * n * n + (size_t)r0 * n, bytes, &bars[sl]);
    };
    if (D > 0 && tid == 0) {
        for (int k = 0; k < D; ++k) mbar_init(&bars[k], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (D > 0 && bytes > 0 && tid == 0)
        for (int t = 1; t <= min(D, T); ++t) issue(t);
    const int first = FWD ? 0 : nc - 1;
    for (int t = 1; t < nc; ++t) {
        const int c = chunk_at(t);
        const double* curg = (t == 1) ? ends + (size_t)first * n : Ug + (size_t)(t - 1) * n;
        long long c0 = TKCLK();
        if (t >= 2) {
            if (tid == 0) {
                const unsigned target = (unsigned)(t - 1) * (unsigned)G;
                unsigned v;
                do {
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(cnt) : "memory");
                } while (v < target);
            }
            __syncthreads();
        }
        long long c1 = TKCLK();
        TKA(8, c1 - c0);
        for (int j = tid; j < n; j += blockDim.x) Us[j] = __ldcg(curg + j);
        __syncthreads();
        long long c2 = TKCLK();
        TKA(11, c2 - c1);
        for (int j = r0 + tid; j < r1; j += blockDim.x) starts[(size_t)c * n + j] = Us[j];
        if (t == nc - 1) break;
        const int sl = D > 0 ? (t - 1) % D : 0;
        if (D > 0 && bytes > 0) mbar_wait(&bars[sl], (unsigned)(((t - 1) / D) & 1));
        c1 = TKCLK();
        TKA(9, c1 - c2);
        const double* src = D > 0 ? sm + sl * slot : M + (size_t)c * n * n + (size_t)r0 * n;
        const double* ec = ends + (size_t)c * n;
        for (int r = r0 + warp; r < r1; r += nw) {
            const double* row = src + (size_t)(r - r0) * n;
            double acc = 0.0;
            for (int k = lane; k < n; k += 32) acc = fma(row[k], Us[k], acc);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) __stcg(Ug + (size_t)t * n + r, ec[r] + acc);
        }
        __syncthreads();
        TKA(10, TKCLK() - c1);
        if (tid == 0) {
            if (D > 0 && bytes > 0 && t + D <= T) issue(t + D);
            __threadfence();
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(cnt) : "memory");
        }
    }
    if (tid == 0) {   // last CTA out resets the counters
        __threadfence();
        const unsigned prev = atomicAdd(cnt + 1, 1u);
        if (prev == (unsigned)G - 1) {
            atomicExch(cnt, 0u);
            atomicExch(cnt + 1, 0u);
        }
    }
}

// out[b][c][r] = in[b][r][c] for count n x n matrices
__global__ void tri_transpose(const double* __restrict__ in, double* __restrict__ out, int n) {
    __shared__ double tile[32][33];
    const size_t off = (size_t)blockIdx.z * n * n;
    const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int gr = by + r, gc = bx + threadIdx.x;
        if (gr < n && gc < n) tile[r][threadIdx.x] = in[off + (size_t)gr * n + gc];
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int gr = bx + r, gc = by + threadIdx.x;
        if (gr < n && gc < n) out[off + (size_t)gr * n + gc] = tile[threadIdx.x][r];
    }
}

static int carry_mode(int n);
// group size of the two-level carry for nc chunks (0: single serial carry).
// At most 9 groups: one 16-CTA cluster per group must be co-resident.
// TK_CARRY_GROUP overrides (0 disables).
static int carry_group(int n, int nc) {
    static int forced = -2;
    if (forced == -2) {
        const char* e = getenv("TK_CARRY_GROUP");
        forced = e ? atoi(e) : -1;
    }
    const int T = nc - 2;   // transitions
    if (forced >= 0) return (forced >= 2 && T >= 2 * forced) ? forced : 0;
    if (carry_mode(n) != 1 || T <= 12) return 0;
    int g = (int)sqrt((double)T);
    const int need = (T + 8) / 9;
    return g < need ? need : g;
}
static int chain_ng(int nc, int G) { return G > 0 ? (nc - 2 + G - 1) / G : 0; }

int32_t tri_chain_chunk_default(int n, int N) {
    const int K = N - 1;
    if (n < 2 || K < 24) return 0;
    if (carry_mode(n) == 1 && K >= 128) {
        // grouped carry: phases A and C stream every chunk propagator (n^2
        // doubles each) once, so fewer, longer chunks than the latency-only
        // optimum (K/2)^(1/3); measured on configs[2] (n=512, K=511): Lc = 12
        // (203 us per substitution) vs 7 (264) and 20 (232)
        int lc = (int)ceil(sqrt(K / 4.0));
        const int need = (K + 147) / 148;
        if (lc < need) lc = need;
        if (lc < 4) lc = 4;
        const int nc = (K + lc - 1) / lc;
        if (carry_group(n, nc) > 0) return lc;
    }
    int lc = (int)ceil(sqrt(K / 2.0));
    const int need = (K + 147) / 148;    // at most one chunk per SM
    if (lc < need) lc = need;
    if (lc < 4) lc = 4;
    return lc;
}
static int chain_nc(int N, int Lc) {
    const int K = N - 1;
    if (Lc <= 0 || K <= 0) return 1;
    return (K + Lc - 1) / Lc;
}
// warp-per-chunk chain with precomputed partition factors (tk_tri_chainw.cu)
int chainw_nodes(int n);
int64_t chainw_len(const tk_level* Lv);
int chainw_factor(const tk_level* Lv, double* facw, cudaStream_t s);
int chainw_launch(const tk_level* Lv, bool fwd, const double* a, const double* facw, double* chain,
                  int Lc, int grid, int cbase, const double* st, double* en, cudaStream_t s);

// P, P^T, ends, starts, U_t, counters | Phi, Phi^T, group ends, group starts
static int64_t chain_prod_base_len(const tk_level* Lv) {
    const int64_t n = Lv->n_u, nc = chain_nc(Lv->n_steps, Lv->chain_chunk);
    const int64_t ng = chain_ng((int)nc, carry_group((int)n, (int)nc));
    const int64_t len = 2 * nc * n * n + 3 * nc * n + 4 + 2 * ng * n * n + 2 * ng * n;
    return (len + 1) & ~(int64_t)1;   // the warp-chain records that follow are TMA sources (16 B)
}
int64_t tri_chain_prod_len(const tk_level* Lv) {
    if (Lv->chain_chunk <= 0) return 0;
    return chain_prod_base_len(Lv) + chainw_len(Lv);
}
// the level's warp-chain records (null: tri_chain_kernel runs the chain)
static double* chainw_records(const tk_level* Lv) {
    if (!Lv->chain_prod || Lv->chain_chunk <= 0 || chainw_len(Lv) == 0) return nullptr;
    if (reinterpret_cast<uintptr_t>(Lv->chain_prod) & 15) return nullptr;
    return Lv->chain_prod + chain_prod_base_len(Lv);
}

// ---------------------------------------------------------------------------
// Record-based local solve: the same block row operation as tri_block, with
// the (u,lam) factorisation read from the interval's precomputed record
// (rhs-only cyclic reduction + dense cut solve) instead of being recomputed.
// Shared memory: f0 f1 fw sv srv (padded node arrays) + one partial-sum row.
// ---------------------------------------------------------------------------
static constexpr int kRecArrays = 5;

template <int NT>
__device__ __forceinline__ void tri_block_rec(const TView& V, int i, const double* b,
                                              const double* x, const double* uprev,
                                              const double* munext, double* out, double omega,
                                              const double* xupd, double* sm) {
    const Lay& L = V.lay;
    const int n = dimn<NT>(V), np = padded(n);
    const int tid = threadIdx.x, nth = blockDim.x;
    const bool has_vm = i >= 1, has_uzl = i < L.N;
    double* f0 = sm;
    double* f1 = sm + np;
    double* fw = sm + 2 * np;
    double* sv = sm + 3 * np;
    double* srv = sm + 4 * np;
    double* part = sm + 5 * np;
    const double kap = V.kappa;
    const double* Qv = (i == L.N) ? V.Ql : V.Qm;
    const double* Qu = (i == L.N - 1) ? V.Ql : V.Qm;
    const double* Qz = V.Qz;
    const double* K = has_uzl ? V.Ki(i, n) : nullptr;
    const double* C = (has_uzl && has_vm) ? V.Ci(i, n) : nullptr;
    const int64_t bs = V.sl.base;
    const int64_t ov = L.off_v(i) - bs, ou = L.off_u(i) - bs, oz = L.off_z(i) - bs,
                  om = L.off_mu(i) - bs, ol = L.off_l(i) - bs;
    for (int j = tid; j < n; j += nth) {
        const int J = PI(j);
        double rv = 0.0, ru = 0.0, rz = 0.0, rm = 0.0, rl = 0.0;
        if (b) {
            if (has_vm) { rv = b[ov + j]; rm = b[om + j]; }
            if (has_uzl) { ru = b[ou + j]; rz = b[oz + j]; rl = b[ol + j]; }
        }
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
        if (has_vm) { sv[J] = -rm; srv[J] = rv; }
        if (has_uzl) { f0[J] = ru; f1[J] = rl - kap * rz; fw[J] = rz; }
    }
    __syncthreads();
    if (!has_uzl) {  // last block (v_N, mu_N): mu = Qv v - r_v
        for (int j = tid; j < n; j += nth) {
            const double dv = sv[PI(j)];
            const double dm = tmv_s(Qv, n, sv, j) - srv[PI(j)];
            out[ov + j] = (xupd ? xupd[ov + j] : 0.0) + omega * dv;
            out[om + j] = (xupd ? xupd[om + j] : 0.0) + omega * dm;
        }
        __syncthreads();
        return;
    }
    if (C) {
        for (int j = tid; j < n; j += nth) f1[PI(j)] -= tmv_s(C, n, sv, j);
        __syncthreads();
    }
    const double* fb = V.fac + (size_t)(i - V.sl.r0) * fac_record(n);
    cr_rhs(n, fb, f0, part, false, fw, V.cr, V.qzw);
    for (int j = tid; j < n; j += nth) {
        const int J = PI(j);
        const double du = f0[J], dl = f1[J];
        const double dz = fw[J] - kap * dl;
        out[ou + j] = (xupd ? xupd[ou + j] : 0.0) + omega * du;
        out[oz + j] = (xupd ? xupd[oz + j] : 0.0) + omega * dz;
        out[ol + j] = (xupd ? xupd[ol + j] : 0.0) + omega * dl;
        if (has_vm) {
            const double dv = sv[J];
            double dm = tmv_s(Qv, n, sv, j) - srv[J];
            if (C) dm += tmtv_s(C, n, f1, j);
            out[ov + j] = (xupd ? xupd[ov + j] : 0.0) + omega * dv;
            out[om + j] = (xupd ? xupd[om + j] : 0.0) + omega * dm;
        }
    }
    __syncthreads();
}

int64_t tri_rec_smem_bytes(int n) { return ((int64_t)kRecArrays * padded(n) + 256) * 8; }

// Parallel over block rows with records: jacobi (x may be null) or D^{-1} b.
template <int NT>
__global__ void __launch_bounds__(256, 2) tri_rows_rec(TView V, const double* __restrict__ b,
                                                       const double* __restrict__ x,
                                                       double* __restrict__ y, double omega) {
    extern __shared__ __align__(16) double sm[];
    const Lay& L = V.lay;
    for (int i = V.sl.r0 + blockIdx.x; i < V.sl.r1; i += gridDim.x) {
        const double* uprev = x ? V.sl.uprev(L, x, i) : nullptr;
        const double* munext = x ? V.sl.munext(L, x, i) : nullptr;
        tri_block_rec<NT>(V, i, b, x, uprev, munext, y, omega, x, sm);
    }
}

// Pass 3 of the substitution with records.
template <bool FWD, int NT>
__global__ void __launch_bounds__(256, 2) tri_rows_rec_cpl(TView V, const double* __restrict__ r,
                                                           const double* __restrict__ chain,
                                                           double* __restrict__ y) {
    extern __shared__ __align__(16) double sm[];
    const Lay& L = V.lay;
    const int n = dimn<NT>(V);
    for (int i = blockIdx.x; i <= L.N; i += gridDim.x) {
        const double* uprev = (FWD && i >= 1) ? chain + (size_t)(i - 1) * n : nullptr;
        const double* munext = (!FWD && i < L.N) ? chain + (size_t)(i + 1) * n : nullptr;
        tri_block_rec<NT>(V, i, r, nullptr, uprev, munext, y, 1.0, nullptr, sm);
    }
}

// Pass 3 of the SGS back half (D-U)^{-1} D w:  y_i = w_i - D_i^{-1} U_i y_{i+1}
// (zero rhs, the chain's mu_{i+1} as the coupling, w as the update base).
template <int NT>
__global__ void __launch_bounds__(256, 2) tri_rows_rec_sgsb(TView V, const double* __restrict__ w,
                                                            const double* __restrict__ chain,
                                                            double* __restrict__ y) {
    extern __shared__ __align__(16) double sm[];
    const Lay& L = V.lay;
    const int n = dimn<NT>(V);
    for (int i = blockIdx.x; i <= L.N; i += gridDim.x) {
        const double* munext = i < L.N ? chain + (size_t)(i + 1) * n : nullptr;
        tri_block_rec<NT>(V, i, nullptr, nullptr, nullptr, munext, y, 1.0, w, sm);
    }
}

// Pass 3: parallel solves with the chain as the continuity coupling.
template <bool FWD, int NT>
__global__ void __launch_bounds__(256, 3) tri_rows_cpl(TView V, const double* __restrict__ r,
                                                       const double* __restrict__ chain,
                                                       double* __restrict__ y) {
    extern __shared__ __align__(16) double sm[];
    const Lay& L = V.lay;
    const int n = dimn<NT>(V);
    for (int i = blockIdx.x; i <= L.N; i += gridDim.x) {
        const double* uprev = (FWD && i >= 1) ? chain + (size_t)(i - 1) * n : nullptr;
        const double* munext = (!FWD && i < L.N) ? chain + (size_t)(i + 1) * n : nullptr;
        tri_block<NT>(V, i, r, nullptr, uprev, munext, y, 1.0, nullptr, sm);
    }
}

#ifdef TK_PROF
extern "C" int tk_debug_prof(long long* out16) {
    return cudaMemcpyFromSymbol(out16, g_tk_prof, sizeof(long long) * 16) == cudaSuccess ? 0 : 2;
}
// span of the grouped-carry launches since the last call (ns): kernel-wide
// last end - first start, last start - first start, CTA 0's own duration, for
// phase A (mode 1) and phase C (mode 2)
extern "C" int tk_debug_span(long long* out6) {
    unsigned long long v[8];
    if (cudaMemcpyFromSymbol(v, g_tk_span, sizeof(v)) != cudaSuccess) return 2;
    for (int m = 0; m < 2; ++m) {
        out6[3 * m + 0] = (long long)(v[4 * m + 1] - v[4 * m + 0]);
        out6[3 * m + 1] = (long long)(v[4 * m + 2] - v[4 * m + 0]);
        out6[3 * m + 2] = (long long)v[4 * m + 3];
    }
    const unsigned long long r[8] = {~0ull, 0ull, 0ull, 0ull, ~0ull, 0ull, 0ull, 0ull};
    return cudaMemcpyToSymbol(g_tk_span, r, sizeof(r)) == cudaSuccess ? 0 : 2;
}
#endif

int64_t tri_fac_len(const tk_level* Lv) {
    const int r0 = Lv->row0;
    const int r1 = Lv->row1 > 0 ? Lv->row1 : Lv->n_steps + 1;
    const int stages = (r1 < Lv->n_steps ? r1 : Lv->n_steps) - r0;
    return (int64_t)(stages > 1 ? stages : 1) * fac_record(Lv->n_u);
}
// chain buffer (N+1)*n; for n too large for the shared-memory factor kernel
// also room for a persistent grid of global node-array slices
int64_t tri_scratch_len(const tk_level* Lv) {
    const int n = Lv->n_u;
    const int64_t chain = (int64_t)(Lv->n_steps + 1) * n;
    const int M = 2 * cut_nodes(n);
    const int64_t fsm = (int64_t)kTriArrays * padded(n) * 8 + (int64_t)(M * 2 * M + M) * 8;
    if (fsm <= 227 * 1024) return chain;
    const int64_t work = (int64_t)148 * 2 * kTriArrays * padded(n);
    return chain > work ? chain : work;
}

int32_t tri_cut_nodes(int n) { return cut_nodes(n); }
int32_t tri_cut_level(int n) { return cut_level(n); }

enum TriApply { T_APPLY = 0, T_APPLY_DIAG = 1, T_RESIDUAL = 2 };

// y = A x, D x, or b - A x; one CTA per block row, threads over nodes.
template <int MODE>
__global__ void tri_apply(TView V, const double* __restrict__ b, const double* __restrict__ x,
                          double* __restrict__ y) {
    const Lay& L = V.lay;
    const int n = V.n;
    const double kap = V.kappa;
    const int64_t bs = V.sl.base;
    for (int i = V.sl.r0 + blockIdx.x; i < V.sl.r1; i += gridDim.x) {
        const bool has_vm = i >= 1, has_uzl = i < L.N;
        const double* Qv = (i == L.N) ? V.Ql : V.Qm;
        const double* Qu = (i == L.N - 1) ? V.Ql : V.Qm;
        const double* K = has_uzl ? V.Ki(i, n) : nullptr;
        const double* C = (has_uzl && has_vm) ? V.Ci(i, n) : nullptr;
        const int64_t ov = L.off_v(i) - bs, ou = L.off_u(i) - bs, oz = L.off_z(i) - bs,
                      om = L.off_mu(i) - bs, ol = L.off_l(i) - bs;
        const double* uprev = (MODE != T_APPLY_DIAG) ? V.sl.uprev(L, x, i) : nullptr;
        const double* munext = (MODE != T_APPLY_DIAG) ? V.sl.munext(L, x, i) : nullptr;
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
    if (n < 2 || n > 1664) return 0;
    return (int64_t)kTriArrays * padded(n) * (int64_t)sizeof(double);
}

// threads per CTA of the record-based rows kernels (TK_REC_THREADS overrides)
static int tri_rec_threads(int n) {
    static int forced = -1;
    if (forced < 0) {
        const char* e = getenv("TK_REC_THREADS");
        forced = e ? atoi(e) : 0;
    }
    if (forced >= 32) return forced;
    int t = (n / 4 + 31) / 32 * 32;
    if (t < 32) t = 32;
    if (t > 128) t = 128;
    return t;
}

static int tri_threads(int n) {
    static int forced = -1;
    if (forced < 0) {
        const char* e = getenv("TK_ROWS_THREADS");
        forced = e ? atoi(e) : 0;
    }
    if (forced >= 32 && forced <= 256) return forced;
    int t = (n / 2 + 31) / 32 * 32;
    if (t < 32) t = 32;
    if (t > 256) t = 256;
    return t;
}

static int tri_chain_threads(int n) {
    static int forced = -1;
    if (forced < 0) {
        const char* e = getenv("TK_CHAIN_THREADS");
        forced = e ? atoi(e) : 0;
    }
    if (forced >= 32) return forced;
    int t = (n / 2 + 31) / 32 * 32;
    if (t < 32) t = 32;
    if (t > 256) t = 256;
    return t;
}

// Launch the chunk carry as one cluster: 16 CTAs (non-portable) when that
// fits, else 8; the row blocks are TMA-staged when they fit in shared memory.
// seg_mode 1/2: the grouped carry's phase A / C (clusters = groups).
static int carry_launch(bool fwd, int n, int nc, const double* M, const double* E, double* S,
                        cudaStream_t s, int seg_mode = 0, int G = 0, double* GE = nullptr,
                        const double* GS = nullptr, const double* Phi = nullptr) {
    static int cs_ok = 0;   // cluster size verified for this process
    auto base_for = [&](int) -> int64_t { return (int64_t)2 * n * 8; };   // U ping-pong
    auto smem_for = [&](int cs) -> int64_t {
        const int64_t rpc = (n + cs - 1) / cs;
        return base_for(cs) + rpc * n * 8;
    };
    const int64_t lim = 227 * 1024 - 1024;
    if (!cs_ok) {
        for (void* f : {(void*)tri_chain_carry<true>, (void*)tri_chain_carry<false>,
                        (void*)tri_chain_carry_seg<true>, (void*)tri_chain_carry_seg<false>,
                        (void*)tri_chain_carry<true, true>, (void*)tri_chain_carry<false, true>,
                        (void*)tri_chain_carry_seg<true, true>,
                        (void*)tri_chain_carry_seg<false, true>}) {
            cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lim);
        }
        cudaGetLastError();
        cs_ok = 8;
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 16; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(16); cfg.blockDim = dim3(1024); cfg.dynamicSmemBytes = (size_t)lim;
        cfg.attrs = at; cfg.numAttrs = 1;
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, (const void*)tri_chain_carry<true>, &cfg) ==
                cudaSuccess && ncl > 0)
            cs_ok = 16;
        cudaGetLastError();
    }
    int cs = cs_ok;
    static int forced = -1;
    if (forced < 0) {
        const char* e = getenv("TK_CARRY_CTAS");
        forced = e ? atoi(e) : 0;
    }
    if (forced == 8 || forced == 16) cs = forced < cs_ok ? forced : cs_ok;
    int64_t smem = smem_for(cs);
    int staged = (n % 2 == 0) && smem <= lim && (smem - base_for(cs)) < (1 << 20);
    // register rows (see carry_loadrow): one row per warp; TK_CARRY_REGS=0 keeps the
    // TMA-staged row blocks
    static const bool regs_ok = [] {
        const char* e = getenv("TK_CARRY_REGS");
        return !(e && e[0] == '0');
    }();
    if (regs_ok && n % 64 == 0 && n <= 32 * kCarryNI && n == cs * 32) staged = 2;
    if (staged != 1) smem = base_for(cs);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    int clusters = 1;
    if (seg_mode) {
        const int ng = chain_ng(nc, G);
        clusters = seg_mode == 1 ? ng : ng - 1;
        if (clusters <= 0) return TK_OK;
    }
    cfg.gridDim = dim3(cs * clusters); cfg.blockDim = dim3(1024); cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = s; cfg.attrs = at; cfg.numAttrs = 1;
    cudaError_t e;
    if (seg_mode) {
        auto k = staged == 2 ? (fwd ? tri_chain_carry_seg<true, true> : tri_chain_carry_seg<false, true>)
                             : (fwd ? tri_chain_carry_seg<true> : tri_chain_carry_seg<false>);
        e = cudaLaunchKernelEx(&cfg, k, n, nc, G, seg_mode, M, E, S, GE, GS, staged, Phi);
        return cuda_status(e, "tri_chain_carry_seg");
    }
    auto k = staged == 2 ? (fwd ? tri_chain_carry<true, true> : tri_chain_carry<false, true>)
                         : (fwd ? tri_chain_carry<true> : tri_chain_carry<false>);
    e = cudaLaunchKernelEx(&cfg, k, n, nc, M, E, S, staged);
    return cuda_status(e, "tri_chain_carry");
}

// carry implementation: 1 = one cluster, 0 = grid-wide.  Default: the
// cluster while its row blocks can be TMA-staged (n <= 640), else the grid
// (bandwidth: n^2 doubles per chunk).  TK_CARRY=cluster|grid overrides.
static int carry_mode(int n) {
    static int m = -1;
    if (m < 0) {
        const char* e = getenv("TK_CARRY");
        m = !e ? 2 : (!strcmp(e, "cluster") ? 1 : 0);
    }
    return m == 2 ? (n <= 640 ? 1 : 0) : m;
}

static int carry_grid_launch(bool fwd, int n, int nc, const double* M, const double* E, double* S,
                             double* Ug, unsigned* cnt, cudaStream_t s) {
    static int nsm = 0;
    if (!nsm) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        if (nsm <= 0) nsm = 148;
        for (void* f : {(void*)tri_chain_carry_grid<true>, (void*)tri_chain_carry_grid<false>})
            cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaGetLastError();
    }
    const int R = (n + nsm - 1) / nsm;
    const int G = (n + R - 1) / R;
    const int64_t slot = (int64_t)R * n * 8;
    int D = (int)((160 * 1024) / slot);
    if (D > kCarryRing) D = kCarryRing;
    if (n % 2) D = 0;                       // TMA needs 16-byte multiples
    const int64_t smem = (int64_t)D * slot + (int64_t)n * 8;
    int Ri = R, Di = D;
    void* args[] = {(void*)&n, (void*)&nc, (void*)&M, (void*)&E, (void*)&S, (void*)&Ug,
                    (void*)&cnt, (void*)&Ri, (void*)&Di};
    const void* f = fwd ? (const void*)tri_chain_carry_grid<true> : (const void*)tri_chain_carry_grid<false>;
    const cudaError_t e = cudaLaunchCooperativeKernel(f, dim3(G), dim3(256), args, (size_t)smem, s);
    return cuda_status(e, "tri_chain_carry_grid");
}

int part_nodes_per_lane(int n);
int part_launch(const tk_level* Lv, int mode, const double* b, const double* x, double* y,
                double omega, const double* chain, cudaStream_t s, double* rc = nullptr,
                const double* ec = nullptr, int opt = 0);
bool part_full_rows(const tk_level* Lv);

// warp-per-row partitioned solves (tk_tri_part.cu) for 32 < n <= 512;
// TK_PART=0 selects the CTA-wide cyclic-reduction kernels instead
static bool use_part(int n) {
    static int on = -1;
    if (on < 0) {
        const char* e = getenv("TK_PART");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    return on && part_nodes_per_lane(n) > 0;
}

template <int NT>
static int tri_launch_t(const tk_level* Lv, int op, const double* b, const double* x, double* y,
                        double omega, cudaStream_t s) {
    TView V(Lv);
    const int n = Lv->n_u;
    const int rows = V.sl.r1 - V.sl.r0;
    const int64_t smem = tri_smem_bytes(n);
    static bool attr_done = false;
    if (!attr_done) {
        const int mx = 227 * 1024;
        cudaFuncSetAttribute(tri_rows<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(tri_rows<NT>, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared);
        cudaFuncSetAttribute(tri_subst<true, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(tri_subst<false, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             mx);
        cudaFuncSetAttribute(tri_factor_kernel<NT, false>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(tri_factor_kernel<NT, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(tri_rows_rec<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(tri_rows_rec<NT>, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared);
        cudaFuncSetAttribute(tri_rows_rec_cpl<true, NT>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(tri_rows_rec_sgsb<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(tri_rows_rec_cpl<false, NT>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(tri_rows_cpl<true, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             mx);
        cudaFuncSetAttribute(tri_rows_cpl<false, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             mx);
        cudaFuncSetAttribute(tri_rows_cpl<true, NT>,
                             cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared);
        cudaFuncSetAttribute(tri_rows_cpl<false, NT>,
                             cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared);
        // the chain kernels also hold two static mbarriers
        const int mxc = mx - 1024;
        cudaFuncSetAttribute(tri_chain_kernel<true, true, false, NT>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, mxc);
        cudaFuncSetAttribute(tri_chain_kernel<false, true, false, NT>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, mxc);
        cudaFuncSetAttribute(tri_chain_kernel<true, false, false, NT>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, mxc);
        cudaFuncSetAttribute(tri_chain_kernel<false, false, false, NT>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, mxc);
        cudaFuncSetAttribute(tri_chain_kernel<true, false, true, NT>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, mxc);
        cudaFuncSetAttribute(tri_chain_kernel<true, false, true, NT>,
                             cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_status(e, "tri: cudaFuncSetAttribute");
        attr_done = true;
    }
    const int th = tri_threads(n);
    const bool fast = Lv->fac != nullptr && Lv->scratch != nullptr;
    if (!Lv->qz_w) {
        set_error("tri family: level is missing qz_w");
        return TK_ERR_ARG;
    }
    // record-based D^{-1} only where the partitioned on-the-fly solve cannot run
    // (n_u > 2048): with 512 rows (configs[2] coarsest) tri_rows_part takes
    // 19 us per pass against 26-29 us for the record-based kernels
    const bool rec = Lv->fac != nullptr && !(Lv->flags & TK_FLAG_ONTHEFLY) &&
                     (!use_part(n) || (Lv->flags & TK_FLAG_RECROWS));
    const int64_t rsm = tri_rec_smem_bytes(n);
    const int rth = tri_rec_threads(n);
    if (!rec && smem == 0 && !use_part(n)) {
        set_error("tri family: n_u=%d needs factor records (tk_subst_factor + qz_w)", n);
        return TK_ERR_UNSUPPORTED;
    }
    switch (op) {
        case 3:  // diag solve
            if (!rec && use_part(n)) return part_launch(Lv, 0, b, nullptr, y, 1.0, nullptr, s);
            if (rec) tri_rows_rec<NT><<<rows, rth, rsm, s>>>(V, b, nullptr, y, 1.0);
            else tri_rows<NT><<<rows, th, smem, s>>>(V, b, nullptr, y, 1.0);
            break;
        case 4:  // jacobi
            if (!rec && use_part(n)) return part_launch(Lv, 0, b, x, y, omega, nullptr, s);
            if (rec) tri_rows_rec<NT><<<rows, rth, rsm, s>>>(V, b, x, y, omega);
            else tri_rows<NT><<<rows, th, smem, s>>>(V, b, x, y, omega);
            break;
        case 10:
        case 11:
        case 14: {
            // 14: second half of the symmetric Gauss-Seidel, d = (D-U)^{-1} D w
            // (smoothers.py:130-152) with w = b: pass 1 would compute
            // D^{-1} (D w) = w, so the chain starts from w itself and pass 3
            // solves with a zero rhs on top of w
            const bool fwd = op == 10;
            const bool sgsb = op == 14;
            if (sgsb && !fast) {
                set_error("sgs back half needs the level's factor records");
                return TK_ERR_UNSUPPORTED;
            }
            if (!fast && smem == 0) {
                set_error("tri family: n_u=%d substitutions need factor records (tk_subst_factor)", n);
                return TK_ERR_UNSUPPORTED;
            }
            if (!fast) {
                if (fwd) tri_subst<true, NT><<<1, th, smem, s>>>(V, b, y);
                else tri_subst<false, NT><<<1, th, smem, s>>>(V, b, y);
                break;
            }
            // pass 1: a = D^{-1} r into y
            if (sgsb) {
            } else if (!rec && use_part(n)) {
                const int rc = part_launch(Lv, 0, b, nullptr, y, 1.0, nullptr, s);
                if (rc) return rc;
            } else if (rec) tri_rows_rec<NT><<<rows, rth, rsm, s>>>(V, b, nullptr, y, 1.0);
            else tri_rows<NT><<<rows, th, smem, s>>>(V, b, nullptr, y, 1.0);
            // pass 2: the chain on the coupling vector (serial, or time-chunked)
            const int cth = tri_chain_threads(n);
            const int np = padded(n);
            const int64_t staged = (int64_t)(2 * (fac_record(n) + n) + 4 * np + 256) * 8;
            const int64_t direct = (int64_t)(4 * np + 256) * 8;
            // TMA bulk copies need 16-byte aligned sources and sizes: n even and
            // even segment offsets (always true for the Burgers layout, nz == nu)
            const bool aligned = (n % 2 == 0) && (Lv->n_z % 2 == 0);
            const bool stg = aligned && staged <= 227 * 1024 - 1024;
            const int64_t csm = stg ? staged : direct;
            double* fac = Lv->fac;
            double* chn = Lv->scratch;
            const int N = Lv->n_steps;
            const bool chunked = Lv->chain_prod != nullptr && Lv->chain_chunk > 0;
            const int Lc = chunked ? Lv->chain_chunk : (N > 1 ? N - 1 : 1);
            const int nc = chain_nc(N, Lc);
            double* P = Lv->chain_prod;
            double* PT = chunked ? P + (size_t)nc * n * n : nullptr;
            double* E = chunked ? PT + (size_t)nc * n * n : nullptr;
            double* S = chunked ? E + (size_t)nc * n : nullptr;
            const double* av = sgsb ? b : y;   // D^{-1} r of pass 1 (or w itself)
            const double* facw = chainw_records(Lv);
            int cw_rc = TK_OK;
            auto chain_launch = [&](int grid, int cbase, const double* st, double* en) {
                if (grid <= 0) return;
                if (facw) {   // one warp per chunk, precomputed partition factors
                    const int e = chainw_launch(Lv, fwd, av, facw, chn, Lc, grid, cbase, st, en, s);
                    if (e) cw_rc = e;
                    return;
                }
                if (stg) {
                    if (fwd) tri_chain_kernel<true, true, false, NT><<<grid, cth, csm, s>>>(V, av, fac, chn, Lc, cbase, st, en);
                    else tri_chain_kernel<false, true, false, NT><<<grid, cth, csm, s>>>(V, av, fac, chn, Lc, cbase, st, en);
                } else {
                    if (fwd) tri_chain_kernel<true, false, false, NT><<<grid, cth, csm, s>>>(V, av, fac, chn, Lc, cbase, st, en);
                    else tri_chain_kernel<false, false, false, NT><<<grid, cth, csm, s>>>(V, av, fac, chn, Lc, cbase, st, en);
                }
            };
            if (!chunked || nc == 1) {
                chain_launch(1, 0, nullptr, nullptr);
            } else {
                chain_launch(nc, 0, nullptr, E);                 // all chunks from zero
                double* Ug = S + (size_t)nc * n;
                unsigned* cnt = (unsigned*)(Ug + (size_t)nc * n);
                const int G = carry_group(n, nc);
                int rc;
                if (G > 0) {   // two-level carry: groups from zero -> group starts -> groups again
                    const int ng = chain_ng(nc, G);
                    double* PhiF = reinterpret_cast<double*>(cnt) + 4;
                    double* PhiT = PhiF + (size_t)ng * n * n;
                    double* GE = PhiT + (size_t)ng * n * n;
                    double* GS = GE + (size_t)ng * n;
                    rc = carry_launch(fwd, n, nc, fwd ? P : PT, E, S, s, 1, G, GE, GS);
                    // phases B + C in one launch (seg mode 3: every cluster runs the
                    // group-start recurrence up to its own group, then its transitions);
                    // TK_CARRY_FUSEB=0: the separate phase-B launch
                    static const bool fuse_b = [] {
                        const char* e = getenv("TK_CARRY_FUSEB");
                        return !(e && e[0] == '0');
                    }();
                    if (fuse_b) {
                        if (!rc && ng >= 2)
                            rc = carry_launch(fwd, n, nc, fwd ? P : PT, E, S, s, 3, G, GE, GS,
                                              fwd ? PhiF : PhiT);
                    } else {
                        if (!rc && ng >= 2) rc = carry_launch(fwd, n, ng, fwd ? PhiF : PhiT, GE, GS, s);
                        if (!rc && ng >= 2)
                            rc = carry_launch(fwd, n, nc, fwd ? P : PT, E, S, s, 2, G, GE, GS);
                    }
                } else {
                    rc = carry_mode(n) == 1
                             ? carry_launch(fwd, n, nc, fwd ? P : PT, E, S, s)
                             : carry_grid_launch(fwd, n, nc, fwd ? P : PT, E, S, Ug, cnt, s);
                }
                if (rc) return rc;
                chain_launch(nc - 1, fwd ? 1 : 0, S, nullptr);   // non-seed chunks again
            }
            if (cw_rc) return cw_rc;
            // pass 3: parallel solves with the chain coupling
            if (sgsb && !rec && use_part(n) && y != b) {   // y = w - D^{-1} U y_{+1}: partitioned rows
                const int rc = part_launch(Lv, 4, nullptr, b, y, 1.0, chn, s);
                if (rc) return rc;
            } else if (sgsb) {
                tri_rows_rec_sgsb<NT><<<rows, rth, rsm, s>>>(V, b, chn, y);
            } else if (rec) {
                if (fwd) tri_rows_rec_cpl<true, NT><<<rows, rth, rsm, s>>>(V, b, chn, y);
                else tri_rows_rec_cpl<false, NT><<<rows, rth, rsm, s>>>(V, b, chn, y);
            } else if (use_part(n)) {
                const int rc = part_launch(Lv, fwd ? 1 : 2, b, nullptr, y, 1.0, chn, s);
                if (rc) return rc;
            } else {
                if (fwd) tri_rows_cpl<true, NT><<<rows, th, smem, s>>>(V, b, chn, y);
                else tri_rows_cpl<false, NT><<<rows, th, smem, s>>>(V, b, chn, y);
            }
            break;
        }
        case 12:  // factor
            if (!Lv->fac) {
                set_error("tk_subst_factor: level has no fac buffer");
                return TK_ERR_ARG;
            }
            {
                const int M = 2 * cut_nodes(n);
                const int64_t gsm = (int64_t)(M * 2 * M + M) * 8;
                const int64_t fsm = (smem ? smem : (int64_t)1 << 40) + gsm;
                const int nst = V.sl.r1 - V.sl.r0 < Lv->n_steps ? V.sl.r1 - V.sl.r0 : Lv->n_steps;
                if (fsm <= 227 * 1024) {
                    tri_factor_kernel<NT, false><<<nst, th, fsm, s>>>(V, Lv->fac, nullptr);
                } else {
                    // node arrays in global scratch (large n): a persistent grid
                    const int64_t per = (int64_t)kTriArrays * padded(n);
                    const int grid = (int)(tri_scratch_len(Lv) / per);
                    if (!Lv->scratch || grid < 1) {
                        set_error("tk_subst_factor: n_u=%d needs the level's scratch buffer", n);
                        return TK_ERR_ARG;
                    }
                    tri_factor_kernel<NT, true><<<grid < nst ? grid : nst, th, gsm, s>>>(
                        V, Lv->fac, Lv->scratch);
                }
            }
            break;
        case 13: {  // chunk propagators Pi_c (c = 1..nc-2) and their transposes
            if (!Lv->fac || !Lv->chain_prod || Lv->chain_chunk <= 0) {
                set_error("tk_chain_prod: needs fac, chain_prod and chain_chunk > 0");
                return TK_ERR_ARG;
            }
            const int N = Lv->n_steps, Lc = Lv->chain_chunk, nc = chain_nc(N, Lc);
            if (double* fw = chainw_records(Lv)) {
                const int e = chainw_factor(Lv, fw, s);
                if (e) return e;
            }
            {
                double* cntp = Lv->chain_prod + 2 * (size_t)nc * n * n + 3 * (size_t)nc * n;
                const cudaError_t e = cudaMemsetAsync(cntp, 0, 4 * sizeof(double), s);
                if (e != cudaSuccess) return cuda_status(e, "tk_chain_prod: memset");
            }
            if (nc <= 2) break;
            double* P = Lv->chain_prod;
            double* PT = P + (size_t)nc * n * n;
            const int cth = tri_chain_threads(n);
            const int64_t direct = (int64_t)(4 * padded(n) + 256) * 8;
            dim3 g(nc - 2, n);
            tri_chain_kernel<true, false, true, NT><<<g, cth, direct, s>>>(V, nullptr, Lv->fac, nullptr, Lc, 1, nullptr, PT);
            dim3 tg((n + 31) / 32, (n + 31) / 32, nc);
            tri_transpose<<<tg, dim3(32, 8), 0, s>>>(PT, P, n);
            const int G = carry_group(n, nc);
            if (G > 0) {   // group propagators Phi_g over chunks [1+gG, (g+1)G] (rows of Phi^T)
                const int ng = chain_ng(nc, G);
                double* PhiF = Lv->chain_prod + 2 * (size_t)nc * n * n + 3 * (size_t)nc * n + 4;
                double* PhiT = PhiF + (size_t)ng * n * n;
                dim3 gg(ng, n);
                tri_chain_kernel<true, false, true, NT><<<gg, cth, direct, s>>>(V, nullptr, Lv->fac, nullptr, Lc, 1, nullptr, PhiT, G);
                dim3 tg2((n + 31) / 32, (n + 31) / 32, ng);
                tri_transpose<<<tg2, dim3(32, 8), 0, s>>>(PhiT, PhiF, n);
            }
            break;
        }
        default: set_error("tri: bad op %d", op); return TK_ERR_ARG;
    }
    return check_launch("tri_rows");
}

static bool use_part(int n);
// y = D^{-1} b (zero-start sweep, omega = 1) and the restricted residual rc
// of tk_residual_restrict_jacobi0 in one pass (tri_rows_part<..., RJ>)
bool tri_jacobi0_restrict_ok(const tk_level* Lv, double omega) {
    const int n = Lv->n_u;
    const bool rec = Lv->fac != nullptr && !(Lv->flags & TK_FLAG_ONTHEFLY) &&
                     (!use_part(n) || (Lv->flags & TK_FLAG_RECROWS));
    // the whole level, or a time slab cut at even rows (the coarse entries fed by
    // the neighbouring slabs' rows: tk_restrict_fix_slab)
    const int r1 = Lv->row1 > 0 ? Lv->row1 : Lv->n_steps + 1;
    const bool slab = (Lv->row0 & 1) == 0 && (r1 == Lv->n_steps + 1 || (r1 & 1) == 0) &&
                      r1 - Lv->row0 >= 2;
    return Lv->family == TK_FAMILY_TRI && omega == 1.0 && !rec && use_part(n) &&
           part_nodes_per_lane(n) > 0 && slab && (Lv->n_steps % 2) == 0 && Lv->n_steps >= 2;
}

// after tk_jacobi0_restrict(_um) on a time slab and the halo exchange of its
// iterate y: the two coarse segments fed by the neighbouring slabs' rows --
// the slab's first coarse mu = -(u of fine row row0 - 1) = -halo_u, its last
// coarse u = -(mu of fine row row1) = -halo_mu
// phase 0: rc = 0 - halo (zero-start sweep); 1: rc = halo (the halos of the sweep's
// INPUT x, before the exchange of its output y); 2: rc = rc - halo (after it):
// phases 1 + 2 give (x - y) at the two segments, as the rows write it in-slab
__global__ void tri_restrict_fix_slab(Lay Lc, int64_t cb, int c0, int c1, bool has_prev,
                                      bool has_next, const double* __restrict__ hu,
                                      const double* __restrict__ hm, double* __restrict__ rc,
                                      int phase) {
    const int n = Lc.nu;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < 2 * n; j += gridDim.x * blockDim.x) {
        double* p = nullptr;
        double h = 0.0;
        if (j < n) {
            if (has_prev) { p = rc + (Lc.off_mu(c0) - cb + j); h = hu[j]; }
        } else if (has_next) {
            p = rc + (Lc.off_u(c1 - 1) - cb + (j - n)); h = hm[j - n];
        }
        if (p) *p = phase == 1 ? h : (phase == 2 ? *p - h : 0.0 - h);
    }
}
int tri_restrict_fix_slab_launch(const tk_level* Lv, double* rc, cudaStream_t s, int phase) {
    const int N = Lv->n_steps, n = Lv->n_u;
    const int r1 = Lv->row1 > 0 ? Lv->row1 : N + 1;
    const bool has_prev = Lv->row0 > 0, has_next = r1 <= N;
    if (!has_prev && !has_next) return TK_OK;
    if ((N & 1) || (Lv->row0 & 1) || (has_next && (r1 & 1)) || (has_prev && !Lv->halo_u) ||
        (has_next && !Lv->halo_mu)) {
        set_error("tk_restrict_fix_slab: slab cut at even rows with its halos");
        return TK_ERR_ARG;
    }
    const Lay Lc(N / 2, n, Lv->n_z);
    const int c0 = Lv->row0 / 2, c1 = has_next ? r1 / 2 : N / 2 + 1;
    tri_restrict_fix_slab<<<(2 * n + 255) / 256, 256, 0, s>>>(Lc, Lc.start(c0), c0, c1, has_prev,
                                                            has_next, Lv->halo_u, Lv->halo_mu, rc,
                                                            phase);
    return check_launch("tri_restrict_fix_slab");
}
int tri_jacobi0_restrict_launch(const tk_level* Lv, const double* b, double omega, double* y,
                                double* rc, cudaStream_t s, int partial) {
    if (!tri_jacobi0_restrict_ok(Lv, omega)) {
        set_error("tk_jacobi0_restrict: level not supported (TRI partitioned rows, whole level, "
                  "even N, omega = 1)");
        return TK_ERR_UNSUPPORTED;
    }
    return part_launch(Lv, 0, b, nullptr, y, omega, nullptr, s, rc, nullptr, partial ? 1 : 0);
}
// one omega = 1 sweep from x (may be null) + its restricted residual
int tri_jacobi_restrict_launch(const tk_level* Lv, const double* b, const double* x, double* y,
                               double* rc, cudaStream_t s) {
    if (!tri_jacobi0_restrict_ok(Lv, 1.0)) {
        set_error("tk_jacobi_restrict: level not supported (TRI partitioned rows, whole level, "
                  "even N)");
        return TK_ERR_UNSUPPORTED;
    }
    return part_launch(Lv, 0, b, x, y, 1.0, nullptr, s, rc, nullptr, 0);
}

// y = D^{-1}(b + (L + U)(x + P ec)): the V-cycle's prolongation fused into
// the omega = 1 post-smoothing sweep (tri_rows_part<..., PR>); only the u and
// mu segments of x are read
bool tri_jacobi_prolong_ok(const tk_level* Lv, double omega) {
    return tri_jacobi0_restrict_ok(Lv, omega) && part_full_rows(Lv);
}
// chalo (time slabs): [previous slab's last coarse (u, lam) | next slab's first
// coarse (v, mu)], 4 n_u doubles
int tri_jacobi_prolong_launch(const tk_level* Lv, const double* b, const double* x,
                              const double* ec, double* y, cudaStream_t s, const double* chalo) {
    if (!tri_jacobi_prolong_ok(Lv, 1.0)) {
        set_error("tk_jacobi_prolong: level not supported (TRI partitioned full rows, whole "
                  "level or slab cut at even rows, even N)");
        return TK_ERR_UNSUPPORTED;
    }
    const bool whole = Lv->row0 == 0 && (Lv->row1 == 0 || Lv->row1 == Lv->n_steps + 1);
    if (!whole && !chalo) {
        set_error("tk_jacobi_prolong: a time slab needs its coarse halos (tk_jacobi_prolong_slab)");
        return TK_ERR_ARG;
    }
    return part_launch(Lv, 0, b, x, y, 1.0, nullptr, s, const_cast<double*>(chalo), ec, 0);
}

int tri_launch(const tk_level* Lv, int op, const double* b, const double* x, double* y,
               double omega, cudaStream_t s) {
    TView V(Lv);
    const int n = Lv->n_u;
    if (Lv->n_z != Lv->n_u) {
        set_error("tri family needs n_z == n_u (got %d, %d)", Lv->n_u, Lv->n_z);
        return TK_ERR_UNSUPPORTED;
    }
    if (op >= 10 && !V.sl.whole(Lv->n_steps)) {
        set_error("block Gauss-Seidel substitution needs the whole level (no time slab)");
        return TK_ERR_ARG;
    }
    const int rows = V.sl.r1 - V.sl.r0;
    if (op == T_APPLY || op == T_APPLY_DIAG || op == T_RESIDUAL) {
        // TK_APPLY_THREADS overrides (experiments)
        static const int th_env = getenv("TK_APPLY_THREADS") ? atoi(getenv("TK_APPLY_THREADS")) : 0;
        const int th = th_env >= 32 ? th_env : (n >= 256 ? 256 : 128);
        const int grid = rows < (1 << 30) ? rows : (1 << 30);
        if (op == T_APPLY) tri_apply<T_APPLY><<<grid, th, 0, s>>>(V, b, x, y);
        else if (op == T_APPLY_DIAG) tri_apply<T_APPLY_DIAG><<<grid, th, 0, s>>>(V, b, x, y);
        else tri_apply<T_RESIDUAL><<<grid, th, 0, s>>>(V, b, x, y);
        return check_launch("tri_apply");
    }
    if (n < 2 || n > 4096) {
        set_error("tri family kernels support 2 <= n_u <= 4096 (got %d)", n);
        return TK_ERR_UNSUPPORTED;
    }
    // compile-time n_u only for the headline size: the kernels behind tri_launch_t
    // (CTA-wide cyclic reduction, record-based rows, the homogeneous chain runs of the
    // set-up) are off the hot path since the partitioned rows and the partition-factor
    // chain took over, and every further size costs ~25 s of build time
    switch (n) {
        case 512: return tri_launch_t<512>(Lv, op, b, x, y, omega, s);
        default: return tri_launch_t<0>(Lv, op, b, x, y, omega, s);
    }
}

}  // namespace tk
