// (included by tk_tri_part.cu and the per-width instantiation units tk_tri_part_w*.cu)
// TRI family: partitioned local KKT solves (one CTA per block row, four
// nodes per thread, everything in registers).
//
// Same block-row operation as tri_block (tk_tri.cu; reference kkt.py:298-389
// DiagonalSolver.solve_all, smoothers.py:61-76 jacobi_apply): residual,
// exact solve of the interval's KKT block, update.  Instead of cyclic
// reduction over all n nodes (one barrier per level, half the threads idle
// after the first), the nodes are partitioned into T = 32W contiguous chunks
// of four, one per thread:
//
//   * phase 1: the thread forms the residual of its chunk in registers from
//     16-byte loads (the vector data of the row was staged into the thread's
//     own shared-memory slots by cp.async while the previous row was solved;
//     the stage data K, C comes from L2, prefetched by a TMA bulk prefetch),
//   * two Thomas sweeps over the chunk's three interior nodes: bottom-up (the
//     first interior node in terms of the two chunk interfaces) and top-down
//     (factors T_k = D'_k^{-1} U_k and D'_k^{-1} kept for the back-substitution),
//   * the T interface nodes (the last node of every chunk) form a symmetric
//     2x2-block tridiagonal system, solved by parallel cyclic reduction with
//     a ping-pong shared exchange (one barrier per step),
//   * a forward rhs sweep with the known left interface and a
//     back-substitution recover the interior; the output is written with
//     16-byte stores.
//
// The scalar system Q_z w = r_z rides along through the same steps.  The grid
// is persistent (two CTAs per SM loop over the block rows).  Nodes >= n pad
// the system to 4T nodes with identity blocks.
#include <cooperative_groups.h>

#include "tk_tri.cuh"

namespace tk {

namespace {

#ifndef TK_PART_CHUNK
#define TK_PART_CHUNK 4          // nodes per thread (even)
#endif
constexpr int kChunk = TK_PART_CHUNK;
#ifndef TK_PART_STAGE
#define TK_PART_STAGE 0          // 1: cp.async staging of the next row's vectors (0: L2 bulk prefetch + a large L1)
#endif
#ifndef TK_PART_MINB
#define TK_PART_MINB 2           // CTAs per SM the W=4 build is register-limited to
#endif
#ifndef TK_PART_MINB3
#define TK_PART_MINB3 3          // the same for the x-free rows (MODE 1/2/3) up to W = 4
#endif
constexpr bool kStage = TK_PART_STAGE != 0;
#ifndef TK_PART_PFD
#define TK_PART_PFD 0            // L2 bulk prefetch distance in rows of this CTA: 0 = the row itself, as
                                 // one burst at its start (with 3 CTAs per SM the other rows hide the
                                 // latency; a row ahead measured equal for the plain sweeps and slower
                                 // for the fused prolongation: 0.352 vs 0.345 ms at n_u = 512, 8.30 vs
                                 // 6.74 ms at n_u = 2048)
#endif
#ifndef TK_PART_SINGLE
#define TK_PART_SINGLE 0         // 1: single PCR exchange buffer for W >= 8 (measured: no gain at n_u = 2048)
#endif
#ifndef TK_PART_EARLY
#define TK_PART_EARLY 0          // 1: issue the output's loads before the interface solve (better while the kernel spilled)
#endif
constexpr unsigned kFull = 0xffffffffu;
constexpr int kPX = 19;          // symmetric PCR: published doubles per row
constexpr int kSgC = 12, kSgN = 12;   // staged chunk arrays / neighbour values per thread
constexpr int kFac = 9;          // per interior node: T_k (4), D'_k^{-1} (3), scalar t_k, 1/d'_k

struct S2 { double a, b, c; };   // symmetric [[a b][b c]]

}  // namespace

template <int W>
struct PartCta {
    static constexpr int T = 32 * W;          // threads = chunks = interface nodes
    static constexpr int P = kChunk * T;      // padded system size
    // TK_PART_SINGLE=1 (W >= 8): ONE exchange buffer with a second barrier per PCR
    // step instead of a ping-pong pair (frees 78 KB for L1 at W = 16; measured
    // equal at n_u = 2048: 6.16 vs 6.14 ms per sweep, so the pair stays)
    static constexpr bool kSingle = TK_PART_SINGLE != 0 && W >= 8 && !kStage;
    static constexpr int64_t smem_bytes() {
        return ((int64_t)((kSingle ? 1 : 2) * kPX + (kStage ? kChunk * kSgC + kSgN : 0)) * T) * 8;
    }
    // resident CTAs per SM the build is register-limited to.  The residual
    // form (MODE 0, ~232 registers): 8 warps per SM.  The x-free rows (MODE
    // 1/2/3): 164 registers for 12 warps per SM up to W = 4 and 128
    // registers for 16 warps per SM at W = 8 / 16 (no spills).
    static constexpr int min_blocks(int mode = 0, int mb = 0) {
        if (mb > 0) return mb;
        if (mode == 0) return (TK_PART_MINB * 4) / W > 1 ? (TK_PART_MINB * 4) / W : 1;
        if (W >= 8) return 16 / W;
        return (TK_PART_MINB3 * 4) / W;
    }
};

// NA consecutive nodes [j0, j0+NA) of segment p + o (zero beyond n), NA even.
// FULL: n is a multiple of the chunk count and every segment is 16-byte aligned.
template <bool FULL, int NA>
__device__ __forceinline__ void ld4(const double* __restrict__ p, int64_t o, int j0, int n,
                                    bool on, double (&r)[NA]) {
    if (!on) {
#pragma unroll
        for (int k = 0; k < NA; ++k) r[k] = 0.0;
        return;
    }
    const double* a = p + o + j0;
    if (FULL || (j0 + NA - 1 < n && ((reinterpret_cast<uintptr_t>(a) & 15) == 0))) {
#pragma unroll
        for (int k = 0; k < NA; k += 2) {
            const double2 u = *reinterpret_cast<const double2*>(a + k);
            r[k] = u.x; r[k + 1] = u.y;
        }
    } else {
#pragma unroll
        for (int k = 0; k < NA; ++k) r[k] = (j0 + k < n) ? a[k] : 0.0;
    }
}
template <bool FULL, int NA>
__device__ __forceinline__ void st4(double* __restrict__ p, int64_t o, int j0, int n,
                                    const double (&r)[NA]) {
    double* a = p + o + j0;
    if (FULL || (j0 + NA - 1 < n && ((reinterpret_cast<uintptr_t>(a) & 15) == 0))) {
#pragma unroll
        for (int k = 0; k < NA; k += 2) *reinterpret_cast<double2*>(a + k) = make_double2(r[k], r[k + 1]);
    } else {
#pragma unroll
        for (int k = 0; k < NA; ++k)
            if (j0 + k < n) a[k] = r[k];
    }
}
// single node j of segment p + o (zero outside [0, n))
__device__ __forceinline__ double ld1(const double* __restrict__ p, int64_t o, int j, int n,
                                      bool on) {
    return (on && j >= 0 && j < n) ? p[o + j] : 0.0;
}

// L2 prefetch of [p, p + len) doubles (TMA bulk prefetch; 16-byte granules)
__device__ __forceinline__ void pf_l2(const double* p, int64_t len) {
    if (!p || len <= 0) return;
    uintptr_t a = reinterpret_cast<uintptr_t>(p) & ~(uintptr_t)15;
    uintptr_t e = (reinterpret_cast<uintptr_t>(p + len) + 15) & ~(uintptr_t)15;
    while (a < e) {
        const uint32_t sz = (uint32_t)((e - a) > (1u << 20) ? (1u << 20) : (e - a));
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(sz) : "memory");
        a += sz;
    }
}

// 1/x without the IEEE slow path: MUFU estimate + two Newton steps
__device__ __forceinline__ double frcp(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}

__device__ __forceinline__ S2 inv_s2f(double a, double b, double c) {
    const double id = frcp(a * c - b * b);
    return {c * id, -b * id, a * id};
}


// cp.async (LDGSTS) staging of the next block row's vector data: every thread
// copies exactly the nodes it reads later into its own slots, so only its own
// wait_group is needed (no barrier).  8-byte copies zero-fill out-of-range nodes.
__device__ __forceinline__ void cpa16(double* dst, const double* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cpa8(double* dst, const double* src, bool on) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(on ? 8 : 0)
                 : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

template <bool FULL>
__device__ __forceinline__ void stage4(double* dst, const double* p, int64_t o, int j0, int n, bool on,
                                       const double* dummy) {
    if (FULL && on) {
#pragma unroll
        for (int k = 0; k < kChunk; k += 2) cpa16(dst + k, p + o + j0 + k);
    } else {
#pragma unroll
        for (int k = 0; k < kChunk; ++k) {
            const bool v = on && j0 + k < n;
            cpa8(dst + k, v ? p + o + j0 + k : dummy, v);
        }
    }
}
__device__ __forceinline__ void stage1(double* dst, const double* p, int64_t o, int j, int n, bool on,
                                       const double* dummy) {
    const bool v = on && j >= 0 && j < n;
    cpa8(dst, v ? p + o + j : dummy, v);
}

// vector sources of block row i (slab-relative offsets; couplings per MODE)
struct RowSrc {
    int64_t ov, ou, oz, om, ol;
    const double* uprev;
    const double* munext;
    bool has_vm, has_uzl;
};
template <int MODE>
__device__ __forceinline__ RowSrc row_src(const TView& V, const double* x, const double* chain, int i) {
    const Lay& L = V.lay;
    const int64_t bs = V.sl.base;
    RowSrc r;
    r.has_vm = i >= 1;
    r.has_uzl = i < L.N;
    r.ov = L.off_v(i) - bs; r.ou = L.off_u(i) - bs; r.oz = L.off_z(i) - bs;
    r.om = L.off_mu(i) - bs; r.ol = L.off_l(i) - bs;
    r.uprev = nullptr;
    r.munext = nullptr;
    if (MODE == 0 || MODE == 3) {
        if (x) { r.uprev = V.sl.uprev(L, x, i); r.munext = V.sl.munext(L, x, i); }
    } else if (MODE == 1) {
        if (i >= 1) r.uprev = chain + (size_t)(i - 1) * V.n;
    } else {
        if (i < L.N) r.munext = chain + (size_t)(i + 1) * V.n;
    }
    return r;
}
// staged arrays (chunk nodes): b v m u z l, x v u z l m, uprev, munext;
// neighbours: b_m, x_v, uprev at j0-1 / j0+4, then x u z l at j0-1 / j0+4
template <bool FULL, int T>
__device__ __forceinline__ void stage_row(double* SG, const RowSrc& r, const double* b, const double* x,
                                          bool hx, int n, int j0) {
    const int t = threadIdx.x;
    constexpr int CT = kChunk * T;
    double* c = SG + kChunk * t;              // [kSgC][kChunk*T]
    double* nb = SG + kSgC * CT + t;          // [kSgN][T]
    const int jL = j0 - 1, jR = j0 + kChunk;
    stage4<FULL>(c + 0 * CT, b, r.ov, j0, n, r.has_vm, b);
    stage4<FULL>(c + 1 * CT, b, r.om, j0, n, r.has_vm, b);
    stage4<FULL>(c + 2 * CT, b, r.ou, j0, n, r.has_uzl, b);
    stage4<FULL>(c + 3 * CT, b, r.oz, j0, n, r.has_uzl, b);
    stage4<FULL>(c + 4 * CT, b, r.ol, j0, n, r.has_uzl, b);
    stage1(nb + 0 * T, b, r.om, jL, n, r.has_vm, b);
    stage1(nb + 1 * T, b, r.om, jR, n, r.has_vm, b);
    const bool up = r.has_vm && r.uprev != nullptr, mn = r.has_uzl && r.munext != nullptr;
    stage4<FULL>(c + 10 * CT, r.uprev, 0, j0, n, up, b);
    stage4<FULL>(c + 11 * CT, r.munext, 0, j0, n, mn, b);
    stage1(nb + 4 * T, r.uprev, 0, jL, n, up, b);
    stage1(nb + 5 * T, r.uprev, 0, jR, n, up, b);
    if (hx) {
        stage4<FULL>(c + 5 * CT, x, r.ov, j0, n, r.has_vm, b);
        stage4<FULL>(c + 6 * CT, x, r.ou, j0, n, r.has_uzl, b);
        stage4<FULL>(c + 7 * CT, x, r.oz, j0, n, r.has_uzl, b);
        stage4<FULL>(c + 8 * CT, x, r.ol, j0, n, r.has_uzl, b);
        stage4<FULL>(c + 9 * CT, x, r.om, j0, n, r.has_vm, b);
        stage1(nb + 2 * T, x, r.ov, jL, n, r.has_vm, b);
        stage1(nb + 3 * T, x, r.ov, jR, n, r.has_vm, b);
        stage1(nb + 6 * T, x, r.ou, jL, n, r.has_uzl, b);
        stage1(nb + 7 * T, x, r.ou, jR, n, r.has_uzl, b);
        stage1(nb + 8 * T, x, r.oz, jL, n, r.has_uzl, b);
        stage1(nb + 9 * T, x, r.oz, jR, n, r.has_uzl, b);
        stage1(nb + 10 * T, x, r.ol, jL, n, r.has_uzl, b);
        stage1(nb + 11 * T, x, r.ol, jR, n, r.has_uzl, b);
    }
    cpa_commit();
}


#ifdef TK_PROF
// per-phase cycles of CTA 0 / thread 0, accumulated over its block rows
static __device__ long long g_part_prof[10];
#define TKPP(slot)                                                          \
    do {                                                                    \
        if (blockIdx.x == 0 && threadIdx.x == 0) {                          \
            const long long c_ = clock64();                                 \
            if (slot > 0) g_part_prof[slot] += c_ - g_part_last;            \
            g_part_last = c_;                                               \
        }                                                                   \
    } while (0)
#ifdef TK_PART_PROF_TU
extern "C" int tk_debug_part_prof(long long* out10) {
    const int e = cudaMemcpyFromSymbol(out10, g_part_prof, sizeof(long long) * 10);
    long long z[10] = {0};
    cudaMemcpyToSymbol(g_part_prof, z, sizeof(z));
    return e == cudaSuccess ? 0 : 2;
}
#endif
#else
#define TKPP(slot) \
    do {           \
    } while (0)
#endif

// MODE 0: Jacobi x + omega D^{-1}(b - A x) (couplings from x through the slab);
// MODE 3: Jacobi with omega = 1, D^{-1}(b + (L + U) x): x enters through the
// coupling segments u_{i-1}, mu_{i+1} only (x == nullptr: D^{-1} b, scaled by omega);
// MODE 1 / 2: pass 3 of the forward / backward substitution (coupling from
// the chain vector, no update);
// MODE 4: pass 3 of the SGS back half (D - U)^{-1} D w (smoothers.py:130-152):
// y_i = w_i - D_i^{-1} U_i y_{i+1}, i.e. MODE 2 with a zero right-hand side
// (b == nullptr) on top of the base vector x = w;
// MB > 0: resident CTAs per SM forced (4: 128 registers) so that a level of
// at most 4 x 148 rows runs as ONE wave instead of two.
//
// Every phase works in chunk order: thread t owns nodes [4t, 4t+4) of every
// segment, loaded with two 16-byte loads per segment (all of a block row's
// loads are independent, so a CTA has its whole row in flight at once) and
// kept in registers through the solve; the neighbours j0-1 and j0+4 come
// from single loads (L1 hits: the adjacent threads load those lines).
//
// CL = 2 (n_u > 1024): a block row spans a 2-CTA cluster; CTA r owns chunks
// [rT, (r+1)T) and the exchanges across the two halves (the neighbour
// chunk's bottom-up results, the interface PCR partners, the left interface
// value and the first lam of the right neighbour) read the peer's shared
// memory (distributed shared memory) after cluster barriers.
//
// RJ (MODE 3, omega == 1, whole level, even N): the sweep also writes the
// restricted residual rc = R (b - A y).  After ANY omega = 1 sweep
// D y = b + (L + U) x, so b - A y = (L + U)(y - x): only the continuity
// couplings of the update y - x (x == nullptr: the zero-start sweep of
// tk_residual_restrict_jacobi0, y itself): row 2c-1 writes -u_{2c} as the coarse mu_c, row 2c writes
// -mu_{2c} as the coarse u_c and the zero v_c, z_{c+1}, lam_{c+1} of coarse
// row c -- the separate restriction kernel and its re-read of y disappear.
//
// TOE (TK_FLAG_TOEPLITZ_W): the weights Qm, Ql, Qz have constant diagonals
// (uniform P1 mass matrices), so each diagonal is one scalar per row instead
// of per-node loads -- same values, same arithmetic, fewer loads/registers.
template <int W, int MODE, bool FULL, int CL, bool RJ, bool TOE, bool PR, int MB, bool SLAB>
__global__ void __launch_bounds__(32 * W, PartCta<W>::min_blocks(MODE, MB))
tri_rows_part(TView V, const double* __restrict__ b, const double* __restrict__ x,
              double* __restrict__ y, double omega, const double* __restrict__ chain,
              double* __restrict__ rc, int opt) {
    using Cf = PartCta<W>;
    constexpr int T = Cf::T;
    constexpr int TT = CL * T;                // interface nodes of a row
    constexpr int NA = kChunk;
    extern __shared__ __align__(16) double sm[];
    const Lay& L = V.lay;
    const int n = FULL ? Cf::P * CL : V.n;
    const int tid = threadIdx.x;
    __builtin_assume(tid < T);
    namespace cgs = cooperative_groups;
    const int rank = CL > 1 ? (int)cgs::this_cluster().block_rank() : 0;
    const int gt = rank * T + tid;            // chunk index within the row
    const int cid = blockIdx.x / CL, ncl = gridDim.x / CL;
    auto csync = [&]() {
        if (CL > 1) cgs::this_cluster().sync();
        else __syncthreads();
    };
    // element k*T of buffer `base` for the chunk with row index g (own or peer smem)
    auto at = [&](const double* base, int g) -> const double* {
        if (CL == 1) return base + g;
        const int o = g / T;
        const double* p = o == rank ? base : cgs::this_cluster().map_shared_rank(base, o);
        return p + (g - o * T);
    };
    const double kap = V.kappa, k2 = kap * kap;
    const double* Qz = V.Qz;
    const bool px = RJ && (opt & 1);   // partial x: only the u and mu segments are stored
    // PR on a time slab: the rc argument carries the coarse halos
    // [previous slab's last coarse (u, lam) | next slab's first coarse (v, mu)]
    const double* chalo = PR ? rc : nullptr;
    double* PX[2] = {sm, Cf::kSingle ? sm : sm + kPX * T};   // PCR ping-pong slots (or one)
    double* XB[1] = {PX[1]};               // exchange 1 (12 per thread; PX[1] is first written at step 2)
    double* SG = sm + (Cf::kSingle ? 1 : 2) * kPX * T;   // staged vector data of the next row [kSgC*4 + kSgN][T]
    double* XO = nullptr;                  // interface solution (a PCR slot)
    double* LAM = nullptr;                 // first lam of every chunk (the other PCR slot)

    const int j0 = kChunk * gt;
    const int jL = j0 - 1, jR = j0 + NA;
#ifdef TK_PROF
    long long g_part_last = 0;
#endif
    const int64_t bs = V.sl.base;
    // constant weights at the chunk nodes (diagonal, super-diagonal)
    // weight diagonal `part` (0 sub, 1 diag, 2 sup) at the chunk nodes
    auto tw = [&](const double* Q, int part, bool on, double (&r)[NA]) {
        if (TOE) {
            const double v = on ? Q[part == 0 ? 1 : part * n] : 0.0;
#pragma unroll
            for (int k = 0; k < NA; ++k) r[k] = v;
        } else {
            ld4<FULL>(Q, part * n, j0, n, on, r);
        }
    };
    // single node j of diagonal `part` (zero outside [0, n))
    auto tw1 = [&](const double* Q, int part, int j) -> double {
        if (TOE) return (j >= 0 && j < n) ? Q[part == 0 ? 1 : part * n] : 0.0;
        return ld1(Q, part * n, j, n, true);
    };
    double qzd[NA], qzs[NA], qzb[NA];
    tw(Qz, 1, true, qzd);
    tw(Qz, 2, true, qzs);
    tw(Qz, 0, true, qzb);
    const double qzsL = tw1(Qz, 2, jL), qzbR = tw1(Qz, 0, jR);

    if (kStage && V.sl.r0 + cid < V.sl.r1)
        stage_row<FULL, T>(SG, row_src<MODE>(V, x, chain, V.sl.r0 + cid), b, x,
                           MODE == 0 && x != nullptr, n, j0);
    for (int i = V.sl.r0 + cid; i < V.sl.r1; i += ncl) {
        if (kStage) cpa_wait();
        const bool has_vm = i >= 1, has_uzl = i < L.N;
        if (gt == 0 && i + TK_PART_PFD * ncl < V.sl.r1) {   // a later row's data -> L2
            const int i2 = i + TK_PART_PFD * ncl;
            if (!kStage) {
                const int64_t q0 = L.start(i2) - bs;
                const int64_t q1 = (i2 == L.N ? L.dim() : L.start(i2 + 1)) - bs;
                if (b) pf_l2(b + q0, q1 - q0);
                if ((MODE == 0 || MODE == 4) && x) pf_l2(x + q0, q1 - q0);
                if (MODE == 3 && x) {   // only the two coupling segments of x
                    pf_l2(V.sl.uprev(L, x, i2), n);
                    pf_l2(V.sl.munext(L, x, i2), n);
                    if (PR) {   // and the coarse segments this row's couplings interpolate
                        const Lay Lp(L.N / 2, n, L.nz);
                        const int p0 = SLAB ? V.sl.r0 / 2 : 0;
                        const int p1 = SLAB ? (V.sl.r1 == L.N + 1 ? L.N / 2 + 1 : V.sl.r1 / 2)
                                            : L.N / 2 + 1;
                        const int64_t pb = SLAB ? Lp.start(p0) : 0;
                        auto pu = [&](int tc) {
                            if (!SLAB || tc - 1 >= p0) pf_l2(chain + (Lp.t_u(tc) - pb), n);
                        };
                        auto pm_ = [&](int tc) {
                            if (!SLAB || tc < p1) pf_l2(chain + (Lp.t_mu(tc) - pb), n);
                        };
                        if (i2 >= 1) {                      // u_t, t = i2
                            const int t = i2;
                            if ((t & 1) == 0 || t == 1) pu(t == 1 ? 1 : t / 2);
                            else { pu((t - 1) / 2); pu((t + 1) / 2); }
                        }
                        if (i2 < L.N) {                     // mu_t, t = i2 + 1
                            const int t = i2 + 1;
                            if ((t & 1) == 0 || t == 1) pm_(t == 1 ? 1 : t / 2);
                            else { pm_((t - 1) / 2); pm_((t + 1) / 2); }
                        }
                    }
                }
            }
            if (i2 < L.N) {
                pf_l2(V.Ki(i2, n), 3 * n);
                if (i2 >= 1) pf_l2(V.Ci(i2, n), 3 * n);
            }
        }
        const double* Qv = (i == L.N) ? V.Ql : V.Qm;
        const double* Qu = (i == L.N - 1) ? V.Ql : V.Qm;
        const double* K = has_uzl ? V.Ki(i, n) : nullptr;
        const double* C = (has_uzl && has_vm) ? V.Ci(i, n) : nullptr;
        const int64_t ov = L.off_v(i) - bs, ou = L.off_u(i) - bs, oz = L.off_z(i) - bs,
                      om = L.off_mu(i) - bs, ol = L.off_l(i) - bs;
        const double* uprev = nullptr;
        const double* munext = nullptr;
        if (MODE == 0 || MODE == 3) {
            if (x) { uprev = V.sl.uprev(L, x, i); munext = V.sl.munext(L, x, i); }
        } else if (MODE == 1) {
            if (i >= 1) uprev = chain + (size_t)(i - 1) * n;
        } else {
            if (i < L.N) munext = chain + (size_t)(i + 1) * n;
        }
        const bool hx = MODE == 0 && x != nullptr;
        const bool hc = C != nullptr;
        const Lay Lc(L.N / 2, n, L.nz);
        // coarse slice of the slab: coarse rows [c0, c1) stored from offset cb
        // (whole level: every coarse row, cb = 0)
        // (SLAB == false: compile-time constants, the whole-level kernels pay nothing)
        const int c0 = SLAB ? V.sl.r0 / 2 : 0;
        const int c1 = SLAB ? (V.sl.r1 == L.N + 1 ? L.N / 2 + 1 : V.sl.r1 / 2) : L.N / 2 + 1;
        const int64_t cb = SLAB ? Lc.start(c0) : 0;
        // PR: the couplings are those of x + P e (e = chain, the coarse
        // correction; multigrid.py:115-132): for the fine time t of the segment,
        // even t adds coarse t/2, t = 1 coarse 1, odd t >= 3 the mean of coarse
        // (t-1)/2 and (t+1)/2 -- the arithmetic of tk_prolong_add
        const double *upa = nullptr, *upb = nullptr, *mna = nullptr, *mnb = nullptr;
        if (PR) {
            static_assert(!PR || (MODE == 3 && !kStage && !RJ), "PR: MODE 3 rows only");
            // coarse u of time tc (coarse row tc - 1; outside the slab: the previous
            // slab's last coarse u) and coarse mu of time tc (coarse row tc; outside:
            // the next slab's first coarse mu); chalo = [prev (u, lam) | next (v, mu)]
            auto cu = [&](int tc) -> const double* {
                return (!SLAB || tc - 1 >= c0) ? chain + (Lc.t_u(tc) - cb) : chalo;
            };
            auto cm = [&](int tc) -> const double* {
                return (!SLAB || tc < c1) ? chain + (Lc.t_mu(tc) - cb) : chalo + 3 * n;
            };
            if (uprev) {          // u_t, t = i
                const int t = i;
                if ((t & 1) == 0 || t == 1) upa = cu(t == 1 ? 1 : t / 2);
                else { upa = cu((t - 1) / 2); upb = cu((t + 1) / 2); }
            }
            if (munext) {         // mu_t, t = i + 1
                const int t = i + 1;
                if ((t & 1) == 0 || t == 1) mna = cm(t == 1 ? 1 : t / 2);
                else { mna = cm((t - 1) / 2); mnb = cm((t + 1) / 2); }
            }
        }
#ifdef TK_PART_PFL1
        // (experiment) the thread's 32 bytes of every segment of the row -> L1 at
        // the row's start, so that the staggered loads below are L1 hits
        if (MODE == 3 && !kStage && FULL) {
            auto p1 = [&](const double* p, int64_t off) {
                if (p) asm volatile("prefetch.global.L1 [%0];" ::"l"(p + off + j0));
            };
            if (has_vm) { p1(b, ov); p1(b, om); }
            if (has_uzl) { p1(b, ou); p1(b, oz); p1(b, ol); }
            p1(uprev, 0); p1(munext, 0);
            p1(upa, 0); p1(upb, 0); p1(mna, 0); p1(mnb, 0);
            if (K) { p1(K, 0); p1(K, n); p1(K, 2 * n); }
            if (C) { p1(C, 0); p1(C, n); p1(C, 2 * n); }
        }
#endif
        // x' = x + P e on the chunk nodes / one node of a coupling segment
        auto pr4 = [&](const double* ca, const double* cb, double (&r)[NA]) {
            if (!PR || !ca) return;
            double a4[NA];
            ld4<FULL>(ca, 0, j0, n, true, a4);
            if (cb) {
                double b4[NA];
                ld4<FULL>(cb, 0, j0, n, true, b4);
#pragma unroll
                for (int k = 0; k < NA; ++k) r[k] = r[k] + 0.5 * (a4[k] + b4[k]);
            } else {
#pragma unroll
                for (int k = 0; k < NA; ++k) r[k] = r[k] + a4[k];
            }
        };
        auto pr1 = [&](const double* ca, const double* cb, int j, double v) -> double {
            if (!PR || !ca || j < 0 || j >= n) return v;
            return cb ? v + 0.5 * (ca[j] + cb[j]) : v + ca[j];
        };
        TKPP(0);

        // ---- phase 1: residual of the chunk in registers
        double f0[NA], f1[NA], fw[NA], pm[NA], kd[NA], ks[NA], kb[NA];
        double ksL, kbR;
        {
            const double* sgc = SG + kChunk * tid;
            const double* sgn = SG + kSgC * kChunk * T + tid;
            auto g4 = [&](int a, double (&r)[NA]) {
                if (kStage) {
#pragma unroll
                    for (int k = 0; k < NA; k += 2) {
                        const double2 u = *reinterpret_cast<const double2*>(sgc + a * kChunk * T + k);
                        r[k] = u.x; r[k + 1] = u.y;
                    }
                    return;
                }
                const bool up = has_vm && uprev != nullptr, mnx = has_uzl && munext != nullptr;
                switch (a) {
                    case 0: ld4<FULL>(b, ov, j0, n, has_vm && MODE != 4, r); break;
                    case 1: ld4<FULL>(b, om, j0, n, has_vm && MODE != 4, r); break;
                    case 2: ld4<FULL>(b, ou, j0, n, has_uzl && MODE != 4, r); break;
                    case 3: ld4<FULL>(b, oz, j0, n, has_uzl && MODE != 4, r); break;
                    case 4: ld4<FULL>(b, ol, j0, n, has_uzl && MODE != 4, r); break;
                    case 5: ld4<FULL>(x, ov, j0, n, has_vm, r); break;
                    case 6: ld4<FULL>(x, ou, j0, n, has_uzl, r); break;
                    case 7: ld4<FULL>(x, oz, j0, n, has_uzl, r); break;
                    case 8: ld4<FULL>(x, ol, j0, n, has_uzl, r); break;
                    case 9: ld4<FULL>(x, om, j0, n, has_vm, r); break;
                    case 10: ld4<FULL>(uprev, 0, j0, n, up, r); break;
                    default: ld4<FULL>(munext, 0, j0, n, mnx, r); break;
                }
            };
            auto g1 = [&](int a) -> double {
                if (kStage) return sgn[a * T];
                const bool up = has_vm && uprev != nullptr;
                switch (a) {
                    case 0: return ld1(b, om, jL, n, has_vm && MODE != 4);
                    case 1: return ld1(b, om, jR, n, has_vm && MODE != 4);
                    case 2: return ld1(x, ov, jL, n, has_vm);
                    case 3: return ld1(x, ov, jR, n, has_vm);
                    case 4: return ld1(uprev, 0, jL, n, up);
                    case 5: return ld1(uprev, 0, jR, n, up);
                    case 6: return ld1(x, ou, jL, n, has_uzl);
                    case 7: return ld1(x, ou, jR, n, has_uzl);
                    case 8: return ld1(x, oz, jL, n, has_uzl);
                    case 9: return ld1(x, oz, jR, n, has_uzl);
                    case 10: return ld1(x, ol, jL, n, has_uzl);
                    default: return ld1(x, ol, jR, n, has_uzl);
                }
            };
            double rv[NA], rm[NA], xv[NA], up[NA];
            g4(0, rv);
            g4(1, rm);
            g4(2, f0);
            g4(3, fw);
            g4(4, f1);
            ld4<FULL>(K, n, j0, n, has_uzl, kd);
            ld4<FULL>(K, 2 * n, j0, n, has_uzl, ks);
            ld4<FULL>(K, 0, j0, n, has_uzl, kb);
            ksL = ld1(K, 2 * n, jL, n, has_uzl);
            kbR = ld1(K, 0, jR, n, has_uzl);
            if (hx) g4(5, xv);
            else {
#pragma unroll
                for (int k = 0; k < NA; ++k) xv[k] = 0.0;
            }
            g4(10, up);
            pr4(upa, upb, up);
            // v at the chunk and its two neighbours
            double vv[NA];
            const double bmL = g1(0), bmR = g1(1);
            const double xvL = hx ? g1(2) : 0.0, xvR = hx ? g1(3) : 0.0;
            const double upL = pr1(upa, upb, jL, g1(4)), upR = pr1(upa, upb, jR, g1(5));
#pragma unroll
            for (int k = 0; k < NA; ++k) vv[k] = -((rm[k] + xv[k]) - up[k]);
            const double vL = -((bmL + xvL) - upL), vR = -((bmR + xvR) - upR);
            if (hx) {
                double xu[NA], xz[NA], xl[NA], xm[NA], mn[NA];
                g4(6, xu);
                g4(7, xz);
                g4(8, xl);
                g4(9, xm);
                g4(11, mn);
                const double xuL = g1(6), xuR = g1(7);
                const double xzL = g1(8), xzR = g1(9);
                const double xlL = g1(10), xlR = g1(11);
                double cd[NA], cs[NA], cb[NA], qvd[NA], qvs[NA], qvb[NA], qud[NA], qus[NA], qub[NA];
                ld4<FULL>(C, n, j0, n, hc, cd);
                ld4<FULL>(C, 2 * n, j0, n, hc, cs);
                ld4<FULL>(C, 0, j0, n, hc, cb);
                const double csL = ld1(C, 2 * n, jL, n, hc), cbR = ld1(C, 0, jR, n, hc);
                tw(Qv, 1, true, qvd);
                tw(Qv, 2, true, qvs);
                tw(Qv, 0, true, qvb);
                tw(Qu, 1, true, qud);
                tw(Qu, 2, true, qus);
                tw(Qu, 0, true, qub);
#pragma unroll
                for (int k = 0; k < NA; ++k) {
                    const int j = j0 + k;
                    const bool lo = j > 0, hi = j < n - 1;
                    const double xvm = k > 0 ? xv[k - 1] : xvL, xvp = k < NA - 1 ? xv[k + 1] : xvR;
                    const double xum = k > 0 ? xu[k - 1] : xuL, xup = k < NA - 1 ? xu[k + 1] : xuR;
                    const double xzm = k > 0 ? xz[k - 1] : xzL, xzp = k < NA - 1 ? xz[k + 1] : xzR;
                    const double xlm = k > 0 ? xl[k - 1] : xlL, xlp = k < NA - 1 ? xl[k + 1] : xlR;
                    const double ksm = k > 0 ? ks[k - 1] : ksL, kbp = k < NA - 1 ? kb[k + 1] : kbR;
                    const double csm = k > 0 ? cs[k - 1] : csL, cbp = k < NA - 1 ? cb[k + 1] : cbR;
                    const double qb = lo ? 1.0 : 0.0, qs = hi ? 1.0 : 0.0;
                    if (has_vm) {
                        double av = (qvd[k] * xv[k] + qb * qvb[k] * xvm + qs * qvs[k] * xvp) - xm[k];
                        if (hc) av += cd[k] * xl[k] + qb * csm * xlm + qs * cbp * xlp;
                        rv[k] -= av;
                    }
                    if (has_uzl) {
                        f0[k] -= (qud[k] * xu[k] + qb * qub[k] * xum + qs * qus[k] * xup) +
                                 (kd[k] * xl[k] + qb * ksm * xlm + qs * kbp * xlp);
                        f0[k] -= mn[k];
                        const double qzz = qzd[k] * xz[k] + qb * qzb[k] * xzm + qs * qzs[k] * xzp;
                        fw[k] -= qzz + kap * (qzd[k] * xl[k] + qb * qzb[k] * xlm + qs * qzs[k] * xlp);
                        double al = (kd[k] * xu[k] + qb * kb[k] * xum + qs * ks[k] * xup) + kap * qzz;
                        if (hc) al += cd[k] * xv[k] + qb * cb[k] * xvm + qs * cs[k] * xvp;
                        f1[k] -= al;
                    }
                }
            } else if (has_uzl && munext) {
                double mn[NA];
                g4(11, mn);
                pr4(mna, mnb, mn);
#pragma unroll
                for (int k = 0; k < NA; ++k) f0[k] -= mn[k];
            }
            // v, the mu part without C^T lam, C v into the lam row
            double qvd[NA], qvs[NA], qvb[NA], cd[NA], cs[NA], cb[NA];
            tw(Qv, 1, has_vm, qvd);
            tw(Qv, 2, has_vm, qvs);
            tw(Qv, 0, has_vm, qvb);
            ld4<FULL>(C, n, j0, n, hc, cd);
            ld4<FULL>(C, 2 * n, j0, n, hc, cs);
            ld4<FULL>(C, 0, j0, n, hc, cb);
#pragma unroll
            for (int k = 0; k < NA; ++k) {
                const int j = j0 + k;
                const bool in = j < n, lo = j > 0, hi = j < n - 1;
                const double vm = (k > 0 ? vv[k - 1] : vL) * (lo ? 1.0 : 0.0);
                const double vp = (k < NA - 1 ? vv[k + 1] : vR) * (hi ? 1.0 : 0.0);
                pm[k] = (qvd[k] * vv[k] + qvb[k] * vm + qvs[k] * vp) - rv[k];
                f1[k] = f1[k] - kap * fw[k];
                if (hc) f1[k] -= cd[k] * vv[k] + cb[k] * vm + cs[k] * vp;
                if (!in) { f0[k] = f1[k] = fw[k] = pm[k] = vv[k] = 0.0; }
            }
            if (has_vm && !px) {
                double o[NA];
                if (hx) {
#pragma unroll
                    for (int k = 0; k < NA; ++k) o[k] = xv[k] + omega * vv[k];
                } else if (MODE == 4) {   // base w (v itself is zero: no rhs, no u coupling)
                    ld4<FULL>(x, ov, j0, n, true, o);
#pragma unroll
                    for (int k = 0; k < NA; ++k) o[k] = o[k] + omega * vv[k];
                } else {
#pragma unroll
                    for (int k = 0; k < NA; ++k) o[k] = omega * vv[k];
                }
                st4<FULL>(y, ov, j0, n, o);
            }
        }
        TKPP(1);
#ifdef TK_PART_PFL1N
        // (experiment) the NEXT row's segments -> L1 once this row's loads are in
        // registers: with one CTA per SM (n_u = 2048) nothing else overlaps a row's
        // load phase
        if (MODE == 3 && !kStage && FULL && i + ncl < V.sl.r1) {
            const int i2 = i + ncl;
            auto p1 = [&](const double* p, int64_t off) {
                if (p) asm volatile("prefetch.global.L1 [%0];" ::"l"(p + off + j0));
            };
            if (i2 >= 1) { p1(b, L.off_v(i2) - bs); p1(b, L.off_mu(i2) - bs); }
            if (i2 < L.N) {
                p1(b, L.off_u(i2) - bs); p1(b, L.off_z(i2) - bs); p1(b, L.off_l(i2) - bs);
                p1(V.Ki(i2, n), 0); p1(V.Ki(i2, n), n); p1(V.Ki(i2, n), 2 * n);
                if (i2 >= 1) { p1(V.Ci(i2, n), 0); p1(V.Ci(i2, n), n); p1(V.Ci(i2, n), 2 * n); }
            }
            if (x) { p1(V.sl.uprev(L, x, i2), 0); p1(V.sl.munext(L, x, i2), 0); }
        }
#endif
        if (RJ && (i & 1) == 0) {   // zeros of coarse row c = i/2: v_c, z_{c+1}, lam_{c+1}
            const int c = i / 2;
            double zr[NA];
#pragma unroll
            for (int k = 0; k < NA; ++k) zr[k] = 0.0;
            if (c >= 1) st4<FULL>(rc, Lc.off_v(c) - cb, j0, n, zr);
            if (c < Lc.N) {
                st4<FULL>(rc, Lc.off_z(c) - cb, j0, n, zr);
                st4<FULL>(rc, Lc.off_l(c) - cb, j0, n, zr);
            }
        }
        if (!has_uzl) {   // last block (v_N, mu_N): mu = Qv v - r_v
            double xm[NA], o[NA];
            ld4<FULL>(x, om, j0, n, hx || MODE == 4, xm);
#pragma unroll
            for (int k = 0; k < NA; ++k) o[k] = xm[k] + omega * pm[k];
            st4<FULL>(y, om, j0, n, o);
            if (RJ) {   // coarse u_{N/2} (coarse row N/2 - 1) = -(mu_N - mu_N of x)
                double xo[NA];
                ld4<FULL>(x, om, j0, n, x != nullptr, xo);
#pragma unroll
                for (int k = 0; k < NA; ++k) o[k] = xo[k] - o[k];
                st4<FULL>(rc, Lc.t_u(i / 2) - cb, j0, n, o);
            }
            continue;
        }

        // ---- chunk solve.  D_k = [[Qu, K], [K, -k^2 Qz]]_kk,
        // U_k = [[Qu_{k,k+1}, K_{k+1,k}], [K_{k,k+1}, -k^2 Qz_{k,k+1}]]; the
        // scalar system has diagonal Qz_kk and coupling Qz_{k,k+1}.
        double qud[NA], qus[NA];
        tw(Qu, 1, true, qud);
        tw(Qu, 2, true, qus);
        const double qusL = tw1(Qu, 2, jL);
        auto Dk = [&](int k, double& a, double& bb, double& c) {
            const bool in = j0 + k < n;
            a = in ? qud[k] : 1.0;
            bb = kd[k];
            c = in ? -k2 * qzd[k] : -1.0;
        };
        auto Uk = [&](int k, double& u0, double& u1, double& u2, double& u3) {   // k = -1..NA-1
            const int j = j0 + k;
            const bool cpl = j >= 0 && j < n - 1;
            u0 = cpl ? (k >= 0 ? qus[k] : qusL) : 0.0;
            u1 = cpl ? (k + 1 < NA ? kb[k + 1] : kbR) : 0.0;
            u2 = cpl ? (k >= 0 ? ks[k] : ksL) : 0.0;
            u3 = cpl ? -k2 * (k >= 0 ? qzs[k] : qzsL) : 0.0;
        };
        auto dzs = [&](int k) -> double { return j0 + k < n ? qzd[k] : 1.0; };
        auto ezs = [&](int k) -> double {   // coupling (j0+k, j0+k+1), k = -1..NA-1
            const int j = j0 + k;
            return (j >= 0 && j < n - 1) ? (k >= 0 ? qzs[k] : qzsL) : 0.0;
        };
        double ul0, ul1, ul2, ul3, ur0, ur1, ur2, ur3;
        Uk(-1, ul0, ul1, ul2, ul3);
        Uk(NA - 1, ur0, ur1, ur2, ur3);
        const double sel = ezs(-1), ser = ezs(NA - 1);

        // step A (bottom-up over the interior): y_0 = iDh (h + H x_R - U_{-1}^T x_L)
        double ha, hb, H00, H01, H10, H11;
        S2 iDh;
        double s_idh, s_hh, s_Hh;
        {
            double da, db, dc;
            Dk(NA - 2, da, db, dc);
            ha = f0[NA - 2];
            hb = f1[NA - 2];
            double u0, u1, u2, u3;
            Uk(NA - 2, u0, u1, u2, u3);
            H00 = -u0; H01 = -u1; H10 = -u2; H11 = -u3;
            double sd = dzs(NA - 2);
            s_hh = fw[NA - 2];
            s_Hh = -ezs(NA - 2);
#pragma unroll
            for (int k = NA - 2; k >= 1; --k) {
                const S2 iv = inv_s2f(da, db, dc);
                Uk(k - 1, u0, u1, u2, u3);
                const double s00 = iv.a * u0 + iv.b * u1, s01 = iv.a * u2 + iv.b * u3;
                const double s10 = iv.b * u0 + iv.c * u1, s11 = iv.b * u2 + iv.c * u3;
                double a, bb, c;
                Dk(k - 1, a, bb, c);
                da = a - (u0 * s00 + u1 * s10);
                db = bb - (u0 * s01 + u1 * s11);
                dc = c - (u2 * s01 + u3 * s11);
                const double nha = f0[k - 1] - (s00 * ha + s10 * hb);
                const double nhb = f1[k - 1] - (s01 * ha + s11 * hb);
                ha = nha; hb = nhb;
                const double n00 = -(s00 * H00 + s10 * H10), n01 = -(s00 * H01 + s10 * H11);
                const double n10 = -(s01 * H00 + s11 * H10), n11 = -(s01 * H01 + s11 * H11);
                H00 = n00; H01 = n01; H10 = n10; H11 = n11;
                const double e = ezs(k - 1);
                const double sb = e * frcp(sd);
                sd = dzs(k - 1) - e * sb;
                s_hh = fw[k - 1] - sb * s_hh;
                s_Hh = -sb * s_Hh;
            }
            iDh = inv_s2f(da, db, dc);
            s_idh = frcp(sd);
        }
        // step B (top-down): T_k, D'_k^{-1} in registers
        double FSr[kFac][NA - 1];   // chunk factors (registers)
        auto fs = [&](int a, int k) -> double& { return FSr[a][k]; };
        double pa, pb, pc, ga, gb, F00, F01, F10, F11, s_dp, s_g, s_F;
        {
            Dk(0, pa, pb, pc);
            ga = f0[0];
            gb = f1[0];
            F00 = -ul0; F01 = -ul2; F10 = -ul1; F11 = -ul3;
            s_dp = dzs(0);
            s_g = fw[0];
            s_F = -sel;
#pragma unroll
            for (int k = 1; k < NA; ++k) {
                const S2 iv = inv_s2f(pa, pb, pc);
                double u0, u1, u2, u3;
                Uk(k - 1, u0, u1, u2, u3);
                const double t00 = iv.a * u0 + iv.b * u2, t01 = iv.a * u1 + iv.b * u3;
                const double t10 = iv.b * u0 + iv.c * u2, t11 = iv.b * u1 + iv.c * u3;
                fs(0, k - 1) = t00; fs(1, k - 1) = t01; fs(2, k - 1) = t10; fs(3, k - 1) = t11;
                fs(4, k - 1) = iv.a; fs(5, k - 1) = iv.b; fs(6, k - 1) = iv.c;
                double a, bb, c;
                Dk(k, a, bb, c);
                pa = a - (u0 * t00 + u2 * t10);
                pb = bb - (u0 * t01 + u2 * t11);
                pc = c - (u1 * t01 + u3 * t11);
                const double nga = f0[k] - (t00 * ga + t10 * gb);
                const double ngb = f1[k] - (t01 * ga + t11 * gb);
                ga = nga; gb = ngb;
                const double n00 = -(t00 * F00 + t10 * F10), n01 = -(t00 * F01 + t10 * F11);
                const double n10 = -(t01 * F00 + t11 * F10), n11 = -(t01 * F01 + t11 * F11);
                F00 = n00; F01 = n01; F10 = n10; F11 = n11;
                const double e = ezs(k - 1);
                const double idp = frcp(s_dp);
                const double tt = e * idp;
                fs(7, k - 1) = tt;
                fs(8, k - 1) = idp;
                s_dp = dzs(k) - e * tt;
                s_g = fw[k] - tt * s_g;
                s_F = -tt * s_F;
            }
        }
        TKPP(2);
        if (kStage && i + ncl < V.sl.r1)   // the next row's vectors -> this thread's slots
            stage_row<FULL, T>(SG, row_src<MODE>(V, x, chain, i + ncl), b, x, hx, n, j0);
        // exchange 1: this chunk's bottom-up results for the previous chunk
        {
            double* E = XB[0];
            E[0 * T + tid] = iDh.a; E[1 * T + tid] = iDh.b; E[2 * T + tid] = iDh.c;
            E[3 * T + tid] = ha; E[4 * T + tid] = hb;
            E[5 * T + tid] = H00; E[6 * T + tid] = H01; E[7 * T + tid] = H10; E[8 * T + tid] = H11;
            E[9 * T + tid] = s_idh; E[10 * T + tid] = s_hh; E[11 * T + tid] = s_Hh;
        }
        csync();
        TKPP(3);
        // step C: symmetric interface rows  C_{l-1}^T X_{l-1} + B_l X_l + C_l X_{l+1} = R_l
        // (B symmetric; the lower coupling is the transposed upper coupling of the
        // row below), block and scalar
        double B00, B01, B11, C00, C01, C10, C11, R0, R1, sB, sC, sR;
        {
            const double* E = at(XB[0], gt + 1 < TT ? gt + 1 : gt);   // last chunk: coupling is zero
            constexpr int nx = 0;
            const double na = E[0 * T + nx], nb = E[1 * T + nx], nc = E[2 * T + nx];
            const double nha = E[3 * T + nx], nhb = E[4 * T + nx];
            const double nH00 = E[5 * T + nx], nH01 = E[6 * T + nx];
            const double nH10 = E[7 * T + nx], nH11 = E[8 * T + nx];
            const double nsi = E[9 * T + nx], nsh = E[10 * T + nx], nsH = E[11 * T + nx];
            const double v00 = ur0 * na + ur1 * nb, v01 = ur0 * nb + ur1 * nc;
            const double v10 = ur2 * na + ur3 * nb, v11 = ur2 * nb + ur3 * nc;
            B00 = pa - (v00 * ur0 + v01 * ur1);
            B01 = pb - (v00 * ur2 + v01 * ur3);
            B11 = pc - (v10 * ur2 + v11 * ur3);
            C00 = v00 * nH00 + v01 * nH10; C01 = v00 * nH01 + v01 * nH11;
            C10 = v10 * nH00 + v11 * nH10; C11 = v10 * nH01 + v11 * nH11;
            R0 = ga - (v00 * nha + v01 * nhb);
            R1 = gb - (v10 * nha + v11 * nhb);
            const double rho = ser * nsi;
            sB = s_dp - ser * rho;
            sC = rho * nsH;
            sR = s_g - rho * nsh;
        }
#if TK_PART_EARLY
        // the output's loads, issued early: their latency overlaps the interface solve
        const bool hxu = (MODE == 0 || MODE == 4) && x != nullptr;
        double oxu[NA], oxz[NA], oxl[NA], oxm[NA], ocd[NA], ocs[NA], ocb[NA];
        ld4<FULL>(x, ou, j0, n, hxu, oxu);
        ld4<FULL>(x, oz, j0, n, hxu, oxz);
        ld4<FULL>(x, ol, j0, n, hxu, oxl);
        ld4<FULL>(x, om, j0, n, hxu && has_vm, oxm);
        ld4<FULL>(C, n, j0, n, hc, ocd);
        ld4<FULL>(C, 2 * n, j0, n, hc, ocs);
        ld4<FULL>(C, 0, j0, n, hc, ocb);
        const double ocsL = ld1(C, 2 * n, jL, n, hc), ocbR = ld1(C, 0, jR, n, hc);
        TKPP(4);
#endif
        if (Cf::kSingle) csync();   // exchange 1 has been read: the buffer is free for the PCR
        // symmetric parallel cyclic reduction (ping-pong slots, one barrier per step).
        // Row l publishes G = C^T B^{-1} C, g = C^T B^{-1} R (for row l+s) and
        // B^{-1}, q = B^{-1} R, P = B^{-1} C (for row l-s).
        {
            int slot = 0;
#pragma unroll
            for (int s = 1; s < TT; s <<= 1) {
                double* E = PX[slot];
                {
                    const S2 iv = inv_s2f(B00, B01, B11);
                    const double q0 = iv.a * R0 + iv.b * R1, q1 = iv.b * R0 + iv.c * R1;
                    const double p00 = iv.a * C00 + iv.b * C10, p01 = iv.a * C01 + iv.b * C11;
                    const double p10 = iv.b * C00 + iv.c * C10, p11 = iv.b * C01 + iv.c * C11;
                    E[0 * T + tid] = C00 * p00 + C10 * p10;
                    E[1 * T + tid] = C00 * p01 + C10 * p11;
                    E[2 * T + tid] = C01 * p01 + C11 * p11;
                    E[3 * T + tid] = C00 * q0 + C10 * q1;
                    E[4 * T + tid] = C01 * q0 + C11 * q1;
                    E[5 * T + tid] = iv.a; E[6 * T + tid] = iv.b; E[7 * T + tid] = iv.c;
                    E[8 * T + tid] = q0; E[9 * T + tid] = q1;
                    E[10 * T + tid] = p00; E[11 * T + tid] = p01;
                    E[12 * T + tid] = p10; E[13 * T + tid] = p11;
                    const double ib = frcp(sB);
                    const double sq = sR * ib, sp = sC * ib;
                    E[14 * T + tid] = sC * sp; E[15 * T + tid] = sC * sq;
                    E[16 * T + tid] = ib; E[17 * T + tid] = sq; E[18 * T + tid] = sp;
                }
                csync();
                if (gt >= s) {
                    const double* Em = at(E, gt - s);
                    constexpr int m = 0;
                    B00 -= Em[0 * T + m]; B01 -= Em[1 * T + m]; B11 -= Em[2 * T + m];
                    R0 -= Em[3 * T + m]; R1 -= Em[4 * T + m];
                    sB -= Em[14 * T + m]; sR -= Em[15 * T + m];
                }
                if (gt + s < TT) {
                    const double* Em = at(E, gt + s);
                    constexpr int m = 0;
                    const double ia = Em[5 * T + m], ib = Em[6 * T + m], ic = Em[7 * T + m];
                    const double q0 = Em[8 * T + m], q1 = Em[9 * T + m];
                    const double p00 = Em[10 * T + m], p01 = Em[11 * T + m];
                    const double p10 = Em[12 * T + m], p11 = Em[13 * T + m];
                    // K = C iB
                    const double k00 = C00 * ia + C01 * ib, k01 = C00 * ib + C01 * ic;
                    const double k10 = C10 * ia + C11 * ib, k11 = C10 * ib + C11 * ic;
                    B00 -= k00 * C00 + k01 * C01;
                    B01 -= k00 * C10 + k01 * C11;
                    B11 -= k10 * C10 + k11 * C11;
                    R0 -= C00 * q0 + C01 * q1;
                    R1 -= C10 * q0 + C11 * q1;
                    const double n00 = -(C00 * p00 + C01 * p10), n01 = -(C00 * p01 + C01 * p11);
                    const double n10 = -(C10 * p00 + C11 * p10), n11 = -(C10 * p01 + C11 * p11);
                    C00 = n00; C01 = n01; C10 = n10; C11 = n11;
                    const double sib = Em[16 * T + m], ssq = Em[17 * T + m], ssp = Em[18 * T + m];
                    sB -= sC * sC * sib;
                    sR -= sC * ssq;
                    sC = -sC * ssp;
                } else {
                    C00 = C01 = C10 = C11 = 0.0;
                    sC = 0.0;
                }
                slot ^= 1;
                if (Cf::kSingle) csync();   // every partner has read this step's values
            }
            const S2 iv = inv_s2f(B00, B01, B11);
            double* E = PX[slot];
            E[tid] = iv.a * R0 + iv.b * R1;
            E[T + tid] = iv.b * R0 + iv.c * R1;
            E[2 * T + tid] = sR * frcp(sB);
            csync();
            XO = E;
            LAM = Cf::kSingle ? E + 4 * T : PX[slot ^ 1];
        }
        TKPP(5);
        const double X0 = XO[tid], X1 = XO[T + tid], sX = XO[2 * T + tid];
        double xl0 = 0.0, xl1 = 0.0, sxl = 0.0;
        if (gt > 0) {
            const double* Xl = at(XO, gt - 1);
            xl0 = Xl[0]; xl1 = Xl[T]; sxl = Xl[2 * T];
        }
        // steps D/E: rhs sweep with the left interface, back-substitution (registers)
        double yu[NA], yl[NA], yw[NA];
        {
            double g0[NA - 1], g1[NA - 1], gs[NA - 1];
            g0[0] = f0[0] - (ul0 * xl0 + ul2 * xl1);
            g1[0] = f1[0] - (ul1 * xl0 + ul3 * xl1);
            gs[0] = fw[0] - sel * sxl;
#pragma unroll
            for (int k = 1; k < NA - 1; ++k) {
                g0[k] = f0[k] - (fs(0, k - 1) * g0[k - 1] + fs(2, k - 1) * g1[k - 1]);
                g1[k] = f1[k] - (fs(1, k - 1) * g0[k - 1] + fs(3, k - 1) * g1[k - 1]);
                gs[k] = fw[k] - fs(7, k - 1) * gs[k - 1];
            }
            yu[NA - 1] = X0; yl[NA - 1] = X1; yw[NA - 1] = sX;
#pragma unroll
            for (int k = NA - 2; k >= 0; --k) {
                const double t00 = fs(0, k), t01 = fs(1, k), t10 = fs(2, k), t11 = fs(3, k);
                const double ia = fs(4, k), ib = fs(5, k), ic = fs(6, k);
                yu[k] = ia * g0[k] + ib * g1[k] - (t00 * yu[k + 1] + t01 * yl[k + 1]);
                yl[k] = ib * g0[k] + ic * g1[k] - (t10 * yu[k + 1] + t11 * yl[k + 1]);
                yw[k] = fs(8, k) * gs[k] - fs(7, k) * yw[k + 1];
            }
        }
        TKPP(6);
        // exchange 3: first lam of every chunk (the C^T lam coupling of the previous chunk)
        {
            LAM[tid] = yl[0];
        }
        csync();
        const double lamR = (gt + 1 < TT) ? *at(LAM, gt + 1) : 0.0;
        TKPP(7);
#if !TK_PART_EARLY
        // the output's loads, issued early: their latency overlaps the interface solve
        const bool hxu = (MODE == 0 || MODE == 4) && x != nullptr;
        double oxu[NA], oxz[NA], oxl[NA], oxm[NA], ocd[NA], ocs[NA], ocb[NA];
        ld4<FULL>(x, ou, j0, n, hxu, oxu);
        ld4<FULL>(x, oz, j0, n, hxu, oxz);
        ld4<FULL>(x, ol, j0, n, hxu, oxl);
        ld4<FULL>(x, om, j0, n, hxu && has_vm, oxm);
        ld4<FULL>(C, n, j0, n, hc, ocd);
        ld4<FULL>(C, 2 * n, j0, n, hc, ocs);
        ld4<FULL>(C, 0, j0, n, hc, ocb);
        const double ocsL = ld1(C, 2 * n, jL, n, hc), ocbR = ld1(C, 0, jR, n, hc);
        TKPP(4);
#endif
        // ---- output (chunk order)
        {
            double o[NA];
#pragma unroll
            for (int k = 0; k < NA; ++k) o[k] = oxu[k] + omega * yu[k];
            st4<FULL>(y, ou, j0, n, o);
            // (a slab's last odd row feeds the NEXT slab's first coarse mu, its first
            // even row the PREVIOUS slab's last coarse u: tk_restrict_fix_slab
            // writes those from the halos of y)
            if (RJ && (i & 1) && (!SLAB || (i + 1) / 2 < c1)) {   // row 2c-1: coarse mu_c = -(u_{2c} - u_{2c} of x)
                double xo[NA];
                ld4<FULL>(x, ou, j0, n, x != nullptr, xo);
#pragma unroll
                for (int k = 0; k < NA; ++k) o[k] = xo[k] - o[k];
                st4<FULL>(rc, Lc.t_mu((i + 1) / 2) - cb, j0, n, o);
            }
            if (!px) {
#pragma unroll
                for (int k = 0; k < NA; ++k) o[k] = oxz[k] + omega * (yw[k] - kap * yl[k]);
                st4<FULL>(y, oz, j0, n, o);
#pragma unroll
                for (int k = 0; k < NA; ++k) o[k] = oxl[k] + omega * yl[k];
                st4<FULL>(y, ol, j0, n, o);
            }
            if (has_vm) {
#pragma unroll
                for (int k = 0; k < NA; ++k) {
                    const int j = j0 + k;
                    const double lm = k > 0 ? yl[k - 1] : xl1;   // lam at j-1 (left interface)
                    const double lp = k < NA - 1 ? yl[k + 1] : lamR;
                    double dm = pm[k];
                    if (hc) {
                        dm += ocd[k] * yl[k];
                        if (j > 0) dm += (k > 0 ? ocs[k - 1] : ocsL) * lm;
                        if (j < n - 1) dm += (k < NA - 1 ? ocb[k + 1] : ocbR) * lp;
                    }
                    o[k] = oxm[k] + omega * dm;
                }
                st4<FULL>(y, om, j0, n, o);
                if (RJ && (i & 1) == 0 && (!SLAB || i / 2 - 1 >= c0)) {   // row 2c: coarse u_c = -(mu_{2c} - mu_{2c} of x)
                    double xo[NA];
                    ld4<FULL>(x, om, j0, n, x != nullptr, xo);
#pragma unroll
                    for (int k = 0; k < NA; ++k) o[k] = xo[k] - o[k];
                    st4<FULL>(rc, Lc.t_u(i / 2) - cb, j0, n, o);
                }
            }
        }
        TKPP(8);
        csync();   // peers are done reading this CTA's exchange slots
        TKPP(9);
    }
}

// ---------------------------------------------------------------------------
// host dispatch
// ---------------------------------------------------------------------------
// warps per CTA and CTAs per row (cluster size).  The x-free rows (modes
// 1/2/3, 128 registers at W >= 8) take up to 16 warps, so n_u <= 2048 is one
// CTA per row; the residual form (mode 0, ~232 registers) takes up to 8 warps
// and splits 1024 < n_u <= 2048 over a 2-CTA cluster.
static int part_wmax(int mode) { return mode == 0 ? 8 : 16; }
static int part_warps(int n, int mode) {
    if (n <= 4 || n > 2 * kChunk * 32 * 8) return 0;
    int w = 1;
    while (kChunk * 32 * w < n && w < part_wmax(mode)) w <<= 1;
    return w;
}
static int part_cluster(int n, int mode) { return n > kChunk * 32 * part_wmax(mode) ? 2 : 1; }

#ifdef TK_PART_MAIN_TU
int part_nodes_per_lane(int n) { return part_warps(n, 0) ? kChunk : 0; }
#endif

template <int W, int MODE, bool FULL, int CL, bool RJ, bool TOE, bool PR, int MB = 0, bool SLAB = false>
static int part_launch_tt(const tk_level* Lv, const double* b, const double* x, double* y,
                          double omega, const double* chain, cudaStream_t s, double* rc, int opt) {
    using Cf = PartCta<W>;
    static int per_sm = 0;
    static int nsm = 0;
    const int64_t smem = Cf::smem_bytes();
    auto kern = tri_rows_part<W, MODE, FULL, CL, RJ, TOE, PR, MB, SLAB>;
    if (!per_sm) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        // shared memory only as large as the resident CTAs need: the rest of the
        // 256 KB unified array stays L1 (stage data, weights and vectors are
        // read through it)
        int carve = cudaSharedmemCarveoutMaxShared;
        if (!kStage) {
            const int64_t need = (int64_t)Cf::min_blocks(MODE, MB) * (smem + 1024);
            carve = (int)((100 * need + 228 * 1024 - 1) / (228 * 1024)) + 1;
            if (carve > 100) carve = 100;
        }
        cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        int per = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 32 * W, (size_t)smem);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_status(e, "tri_rows_part: attributes");
        if (per < 1) {
            set_error("tri_rows_part<%d>: does not fit on an SM (%lld B smem)", W, (long long)smem);
            return TK_ERR_CUDA;
        }
        per_sm = per;
    }
    TView V(Lv);
    const int rows = V.sl.r1 - V.sl.r0;
    int clusters = rows;
    const int cap = nsm * per_sm / CL;
    if (clusters > cap) clusters = cap;
    if (CL == 1) {
        kern<<<clusters, 32 * W, smem, s>>>(V, b, x, y, omega, chain, rc, opt);
        return check_launch("tri_rows_part");
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(clusters * CL); cfg.blockDim = dim3(32 * W); cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = s; cfg.attrs = at; cfg.numAttrs = 1;
    return cuda_status(cudaLaunchKernelEx(&cfg, kern, V, b, x, y, omega, chain, rc, opt),
                       "tri_rows_part (cluster)");
}

static inline bool level_whole(const tk_level* Lv) {
    return Lv->row0 == 0 && (Lv->row1 == 0 || Lv->row1 == Lv->n_steps + 1);
}

// TOE only for FULL rows (every chunk inside the level, so the masked
// boundary entries of the stored diagonals are never needed)
template <int W, int MODE, bool FULL, int CL, bool RJ = false, bool PR = false>
static int part_launch_t(const tk_level* Lv, const double* b, const double* x, double* y,
                         double omega, const double* chain, cudaStream_t s, double* rc = nullptr,
                         int opt = 0) {
    if (FULL && (Lv->flags & TK_FLAG_TOEPLITZ_W)) {
        if (W == 4 && MODE != 0 && !RJ && !PR) {
            // a short level (the coarsest one: 513 rows at configs[2]): 4 CTAs per SM
            // hold every row at once; 3 per SM would run 444 rows, then 69
            static int nsm = 0;
            if (!nsm) {
                int dev = 0;
                cudaGetDevice(&dev);
                cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
            }
            const int r1 = Lv->row1 > 0 ? Lv->row1 : Lv->n_steps + 1;
            const int rows = r1 - Lv->row0;
            if (rows > 3 * nsm && rows <= 4 * nsm)
                return part_launch_tt<W, MODE, FULL, CL, RJ, FULL, PR, (W == 4 && MODE != 0 && !RJ && !PR) ? 4 : 0>(
                    Lv, b, x, y, omega, chain, s, rc, opt);
        }
        if ((RJ || PR) && !level_whole(Lv))   // time slab: the coarse slice / coarse halos
            return part_launch_tt<W, MODE, FULL, CL, RJ, FULL, PR, 0, RJ || PR>(Lv, b, x, y, omega, chain,
                                                                                s, rc, opt);
        return part_launch_tt<W, MODE, FULL, CL, RJ, FULL, PR>(Lv, b, x, y, omega, chain, s, rc, opt);
    }
    if ((RJ || PR) && !level_whole(Lv))
        return part_launch_tt<W, MODE, FULL, CL, RJ, false, PR, 0, RJ || PR>(Lv, b, x, y, omega, chain, s,
                                                                             rc, opt);
    return part_launch_tt<W, MODE, FULL, CL, RJ, false, PR>(Lv, b, x, y, omega, chain, s, rc, opt);
}


// the launches of one row width (WW warps per CTA, CC CTAs per row); -1: not this width.
// Each width is instantiated in its own translation unit (tk_tri_part_w*.cu) so that
// the library builds in parallel.
template <int WW, int CC>
int part_dispatch_x(const tk_level* Lv, int mode, bool full, const double* b, const double* x,
                    double* y, double omega, const double* chain, cudaStream_t s, double* rc,
                    const double* ec, int opt) {
    if (ec) {   // rc: the coarse halos of a time slab (or null)
        if (full) return part_launch_t<WW, 3, true, CC, false, true>(Lv, b, x, y, omega, ec, s, rc);
        return part_launch_t<WW, 3, false, CC, false, true>(Lv, b, x, y, omega, ec, s, rc);
    }
    if (rc) {
        if (full) return part_launch_t<WW, 3, true, CC, true>(Lv, b, x, y, omega, chain, s, rc, opt);
        return part_launch_t<WW, 3, false, CC, true>(Lv, b, x, y, omega, chain, s, rc, opt);
    }
    if (full) {
        if (mode == 3) return part_launch_t<WW, 3, true, CC>(Lv, b, x, y, omega, chain, s);
        if (mode == 1) return part_launch_t<WW, 1, true, CC>(Lv, b, x, y, omega, chain, s);
        if (mode == 2) return part_launch_t<WW, 2, true, CC>(Lv, b, x, y, omega, chain, s);
        if (mode == 4) return part_launch_t<WW, 4, true, CC>(Lv, b, x, y, omega, chain, s);
    } else {
        if (mode == 3) return part_launch_t<WW, 3, false, CC>(Lv, b, x, y, omega, chain, s);
        if (mode == 1) return part_launch_t<WW, 1, false, CC>(Lv, b, x, y, omega, chain, s);
        if (mode == 2) return part_launch_t<WW, 2, false, CC>(Lv, b, x, y, omega, chain, s);
        if (mode == 4) return part_launch_t<WW, 4, false, CC>(Lv, b, x, y, omega, chain, s);
    }
    return -1;
}
template <int WW, int CC>
int part_dispatch_r(const tk_level* Lv, bool full, const double* b, const double* x, double* y,
                    double omega, const double* chain, cudaStream_t s) {
    if (full) return part_launch_t<WW, 0, true, CC>(Lv, b, x, y, omega, chain, s);
    return part_launch_t<WW, 0, false, CC>(Lv, b, x, y, omega, chain, s);
}

}  // namespace tk
