// TRI family: the serial-in-time coupling chain of the block Gauss-Seidel
// substitutions (reference smoothers.py:79-109 _forward_subst /
// _backward_subst: delta_i = D_i^{-1}(r_i + coupling(delta_{i-1}))), one WARP
// per time chunk.
//
// The chain is the recurrence on the n_u coupling vector
//   FWD: u_i  = a_i + P_u   D_i^{-1} E_lam (-C_i u_{i-1})
//   BWD: mu_i = a_i + C_i^T P_lam D_i^{-1} E_u (-mu_{i+1})
// (a = D^{-1} r from pass 1).  Every step is one rhs-only solve of the
// interval's symmetric 2x2-block tridiagonal (u, lam) system
//   [[Q_u, K^T], [K, -kappa^2 Q_z]],
// so its latency is the latency of the whole substitution.  tri_chain_kernel
// (tk_tri.cu) runs it as CTA-wide cyclic reduction: 2 log2(n) barrier-separated
// levels, ~3.4 us per interval at n_u = 512.  Here the interval is solved by a
// partition method whose every coefficient is precomputed per interval
// (tk_chain_prod): thread t owns NA consecutive nodes, the last one being
// interface t, and a step is
//   two independent Thomas rhs sweeps over the chunk (top-down g_k,
//   bottom-up h_k; register recurrences of 2x2 mat-vecs),
//   R_t = g_last - V_t h_0(t+1)                            (one exchange),
//   log2(T) rhs-only parallel-cyclic-reduction steps on the T interface
//   unknowns, R_t -= alpha_t R_{t-s} + gamma_t R_{t+s}      (one exchange each),
//   X_t = Binv_t R_t, and the back-substitution
//   x_k = Di_k g_k + G_k X_{t-1} - T_k x_{k+1}              (one exchange).
// With T = 32 every exchange is a shared-memory round trip fenced by
// __syncwarp: no CTA barrier in the loop (n_u = 512 runs two warps of 8 nodes
// per thread: 3300 cycles per interval against 4200 for one warp of 16 and
// ~6700 for tri_chain_kernel; a step is bound by the latency of its ~500
// dependent-ish fp64 instructions per warp, not by the record traffic --
// tools/cw_phases.py).  The next interval's record (all
// coefficients in [slot][T] order: conflict-free 16-byte shared loads) is
// TMA bulk-copied into the other half of a double buffer while the current
// interval is solved.
#include "tk_tri.cuh"

namespace tk {

namespace {

struct M2 { double a, b, c, d; };   // [[a b][c d]]
__device__ __forceinline__ M2 m2(double a, double b, double c, double d) { return {a, b, c, d}; }
__device__ __forceinline__ M2 inv2(const M2& m) {
    const double id = 1.0 / (m.a * m.d - m.b * m.c);
    return {m.d * id, -m.b * id, -m.c * id, m.a * id};
}
__device__ __forceinline__ M2 mul(const M2& x, const M2& y) {
    return {x.a * y.a + x.b * y.c, x.a * y.b + x.b * y.d, x.c * y.a + x.d * y.c, x.c * y.b + x.d * y.d};
}
__device__ __forceinline__ M2 tr(const M2& x) { return {x.a, x.c, x.b, x.d}; }
__device__ __forceinline__ M2 sub(const M2& x, const M2& y) { return {x.a - y.a, x.b - y.b, x.c - y.c, x.d - y.d}; }
__device__ __forceinline__ M2 neg(const M2& x) { return {-x.a, -x.b, -x.c, -x.d}; }

// record layout, doubles per thread (see the file comment); every entry is a
// 4-double group (2 x double2) except the two edge coefficients at the end
__host__ __device__ constexpr int cw_oT(int) { return 0; }
__host__ __device__ constexpr int cw_oDi(int NA) { return 4 * (NA - 1); }
__host__ __device__ constexpr int cw_oG(int NA) { return 8 * (NA - 1); }
__host__ __device__ constexpr int cw_oS(int NA) { return 12 * (NA - 1); }
__host__ __device__ constexpr int cw_oV(int NA) { return 12 * (NA - 1) + 4 * (NA - 2); }
__host__ __device__ constexpr int cw_oP(int NA) { return cw_oV(NA) + 4; }
__host__ __device__ constexpr int cw_oB(int NA, int LT) { return cw_oP(NA) + 8 * LT; }
__host__ __device__ constexpr int cw_oC(int NA, int LT) { return cw_oB(NA, LT) + 4; }
__host__ __device__ constexpr int cw_oE(int NA, int LT) { return cw_oC(NA, LT) + 4 * NA; }
__host__ __device__ constexpr int cw_slots(int NA, int LT) { return cw_oE(NA, LT) + 4; }

__device__ __forceinline__ unsigned s_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(s_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mb_expect(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(s_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
        ::"r"(s_u32(dst)), "l"(src), "r"(bytes), "r"(s_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred P1;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        " @!P1 bra WAIT_%=;\n}\n" ::"r"(s_u32(bar)), "r"(parity)
        : "memory");
}

template <int T>
__device__ __forceinline__ void bsync() {
    if (T == 32) __syncwarp();
    else __syncthreads();
}

// store / load a 4-double group at slot `s` of thread t ([slot/2][T] double2)
template <int T>
__device__ __forceinline__ void st4g(double* rec, int s, int t, double a, double b, double c, double d) {
    double2* r2 = reinterpret_cast<double2*>(rec);
    r2[(s >> 1) * T + t] = make_double2(a, b);
    r2[((s >> 1) + 1) * T + t] = make_double2(c, d);
}

#ifdef TK_PROF
// cycles of chunk 1 / thread 0: [0] steps, [1] total, [2] waiting for the record, [3] rhs +
// sweeps, [4] interface, [5] back-substitution + output
__device__ long long g_cw_prof[8];
#define CWP(slot, c0)                                                      \
    do {                                                                   \
        if (blockIdx.x == 1 && threadIdx.x == 0) {                         \
            const long long c_ = clock64();                                \
            g_cw_prof[slot] += c_ - c0;                                    \
            c0 = c_;                                                       \
        }                                                                  \
    } while (0)
#else
#define CWP(slot, c0) \
    do {              \
    } while (0)
#endif

}  // namespace

#ifdef TK_PROF
extern "C" int tk_debug_cw_prof(long long* out8) {
    const int e = cudaMemcpyFromSymbol(out8, g_cw_prof, sizeof(long long) * 8);
    long long z[8] = {0};
    cudaMemcpyToSymbol(g_cw_prof, z, sizeof(z));
    return e == cudaSuccess ? 0 : 2;
}
#endif

// ---------------------------------------------------------------------------
// factorisation: one CTA of T threads per interval i = 1..N-1
// ---------------------------------------------------------------------------
template <int NA, int T>
__global__ void __launch_bounds__(T) tri_chainw_factor(TView V, double* __restrict__ facw) {
    constexpr int LT = ilog2(T);
    constexpr int SL = cw_slots(NA, LT);
    __shared__ M2 sA[T], sB[T], sC[T];
    const Lay& L = V.lay;
    const int n = V.n, N = L.N;
    const int t = threadIdx.x;
    const int i = 1 + blockIdx.x;
    if (i > N - 1) return;
    double* rec = facw + (size_t)i * SL * T;
    const double* Qu = (i == N - 1) ? V.Ql : V.Qm;
    const double* K = V.Ki(i, n);
    const double* Cm = V.Ci(i, n);
    const double* Qz = V.Qz;
    const double k2 = V.kappa * V.kappa;
    auto Dn = [&](int j) -> M2 {
        if (j >= n) return m2(1.0, 0.0, 0.0, 1.0);
        return m2(Qu[n + j], K[n + j], K[n + j], -k2 * Qz[n + j]);
    };
    auto Un = [&](int j) -> M2 {   // coupling of node j to node j+1
        if (j < 0 || j + 1 >= n) return m2(0.0, 0.0, 0.0, 0.0);
        return m2(Qu[2 * n + j], K[j + 1], K[2 * n + j], -k2 * Qz[2 * n + j]);
    };
    const int j0 = NA * t;
    // top-down: D'_k, T_k = D'_k^{-1} U_k, F_k (coupling to the left interface)
    M2 Dp = Dn(j0);
    M2 F = neg(tr(Un(j0 - 1)));
#pragma unroll
    for (int k = 0; k < NA - 1; ++k) {
        const M2 Di = inv2(Dp);
        const M2 U = Un(j0 + k);
        const M2 Tk = mul(Di, U);
        const M2 G = mul(Di, F);
        st4g<T>(rec, cw_oT(NA) + 4 * k, t, Tk.a, Tk.b, Tk.c, Tk.d);
        st4g<T>(rec, cw_oDi(NA) + 4 * k, t, Di.a, Di.b, Di.c, Di.d);
        st4g<T>(rec, cw_oG(NA) + 4 * k, t, G.a, G.b, G.c, G.d);
        Dp = sub(Dn(j0 + k + 1), mul(tr(U), Tk));
        F = neg(mul(tr(Tk), F));
    }
    // bottom-up over the interior: S_k = D''_{k+1}^{-1} U_k^T, H_k (coupling to the own interface)
    M2 Dpp = Dn(j0 + NA - 2);
    M2 H = neg(Un(j0 + NA - 2));
#pragma unroll
    for (int k = NA - 3; k >= 0; --k) {
        const M2 U = Un(j0 + k);
        const M2 Sk = mul(inv2(Dpp), tr(U));
        st4g<T>(rec, cw_oS(NA) + 4 * k, t, Sk.a, Sk.b, Sk.c, Sk.d);
        Dpp = sub(Dn(j0 + k), mul(U, Sk));
        H = neg(mul(tr(Sk), H));
    }
    sA[t] = inv2(Dpp);   // iD of this chunk's first node
    sB[t] = H;           // H_0
    __syncthreads();
    // interface row t:  A X_{t-1} + B X_t + C X_{t+1} = R_t
    const M2 Ur = Un(j0 + NA - 1);
    M2 Vm = m2(0.0, 0.0, 0.0, 0.0), B = Dp, C = m2(0.0, 0.0, 0.0, 0.0);
    if (t < T - 1) {
        Vm = mul(Ur, sA[t + 1]);
        B = sub(Dp, mul(Vm, tr(Ur)));
        C = mul(Vm, sB[t + 1]);
    }
    M2 A = neg(F);
    st4g<T>(rec, cw_oV(NA), t, Vm.a, Vm.b, Vm.c, Vm.d);
    __syncthreads();
    // parallel cyclic reduction of the interface system (coefficients only)
#pragma unroll
    for (int l = 0; l < LT; ++l) {
        const int s = 1 << l;
        sA[t] = A; sB[t] = inv2(B); sC[t] = C;
        __syncthreads();
        M2 al = m2(0.0, 0.0, 0.0, 0.0), ga = m2(0.0, 0.0, 0.0, 0.0);
        M2 Bn = B, An = m2(0.0, 0.0, 0.0, 0.0), Cn = m2(0.0, 0.0, 0.0, 0.0);
        if (t >= s) {
            al = mul(A, sB[t - s]);
            Bn = sub(Bn, mul(al, sC[t - s]));
            An = neg(mul(al, sA[t - s]));
        }
        if (t + s < T) {
            ga = mul(C, sB[t + s]);
            Bn = sub(Bn, mul(ga, sA[t + s]));
            Cn = neg(mul(ga, sC[t + s]));
        }
        st4g<T>(rec, cw_oP(NA) + 8 * l, t, al.a, al.b, al.c, al.d);
        st4g<T>(rec, cw_oP(NA) + 8 * l + 4, t, ga.a, ga.b, ga.c, ga.d);
        A = An; B = Bn; C = Cn;
        __syncthreads();
    }
    const M2 Bi = inv2(B);
    st4g<T>(rec, cw_oB(NA, LT), t, Bi.a, Bi.b, Bi.c, Bi.d);
    // C_i diagonals at the chunk nodes (sub, diag, sup) and the two edge coefficients
#pragma unroll
    for (int k = 0; k < NA; ++k) {
        const int j = j0 + k;
        const bool in = j < n;
        st4g<T>(rec, cw_oC(NA, LT) + 4 * k, t, in ? Cm[j] : 0.0, in ? Cm[n + j] : 0.0,
                in ? Cm[2 * n + j] : 0.0, 0.0);
    }
    {
        const int jl = j0 - 1, jr = j0 + NA;
        double2* r2 = reinterpret_cast<double2*>(rec);
        r2[(cw_oE(NA, LT) >> 1) * T + t] =
            make_double2((jl >= 0 && jl < n) ? Cm[2 * n + jl] : 0.0, jr < n ? Cm[jr] : 0.0);
    }
}

// ---------------------------------------------------------------------------
// the chain over the steps of one time chunk (one CTA of T threads per chunk;
// the interface of tri_chain_kernel<FWD, STAGED, false>)
// ---------------------------------------------------------------------------
template <bool FWD, int NA, int T>
__global__ void __launch_bounds__(T, 1)
    tri_chainw_kernel(TView V, const double* __restrict__ a, const double* __restrict__ facw,
                      double* __restrict__ chain, int Lc, int cbase,
                      const double* __restrict__ starts, double* __restrict__ ends) {
    constexpr int LT = ilog2(T);
    constexpr int SL = cw_slots(NA, LT);
    constexpr int REC = SL * T;               // doubles per interval record
    extern __shared__ __align__(16) double sm[];
    __shared__ __align__(8) uint64_t bars[2];
    double2* xH = reinterpret_cast<double2*>(sm + 2 * REC);   // exchange arrays [T] each
    double2* xP[2] = {xH + T, xH + 2 * T};
    double2* xX = xH + 3 * T;
    double2* xE = xH + 4 * T;
    const Lay& L = V.lay;
    const int n = V.n, N = L.N;
    const int t = threadIdx.x;
    const int K = N - 1;
    const int c = cbase + blockIdx.x;
    const int lo = c * Lc, hi = min(K, lo + Lc);
    const int k0 = FWD ? lo : K - hi, k1 = FWD ? hi : K - lo;
    const bool seed = k0 == 0;
    auto blk = [&](int k) { return FWD ? 1 + k : N - 1 - k; };
    auto aseg = [&](int i) { return a + (FWD ? L.off_u(i) : L.off_mu(i)); };
    const int i0 = FWD ? 0 : N;
    const double* s0 = seed ? aseg(i0) : (starts ? starts + (size_t)c * n : nullptr);
    const int j0 = NA * t;
    double w[NA];                              // the incoming coupling vector at the chunk nodes
#pragma unroll
    for (int k = 0; k < NA; ++k) w[k] = (s0 && j0 + k < n) ? s0[j0 + k] : 0.0;
    if (seed) {
#pragma unroll
        for (int k = 0; k < NA; ++k)
            if (j0 + k < n) chain[(size_t)i0 * n + j0 + k] = w[k];
    }
    if (k0 >= k1) return;
    if (t == 0) {
        mb_init(&bars[0], 1);
        mb_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    auto prefetch = [&](int k) {
        const int tt = k - k0;
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        mb_expect(&bars[tt & 1], (unsigned)(REC * sizeof(double)));
        tma_load(sm + (tt & 1) * REC, facw + (size_t)blk(k) * REC, (unsigned)(REC * sizeof(double)),
                 &bars[tt & 1]);
    };
    if (t == 0) prefetch(k0);
    double* eout = ends ? ends + (size_t)c * n : nullptr;
    for (int k = k0; k < k1; ++k) {
        const int tt = k - k0;
        const int i = blk(k);
        bsync<T>();                            // every lane is done with the other buffer
        if (t == 0 && k + 1 < k1) prefetch(k + 1);
        // a_i at the chunk nodes: issued now, consumed after the solve
        double av[NA];
        {
            const double* as = aseg(i) + j0;
#pragma unroll
            for (int q = 0; q < NA; q += 2) {
                if (j0 + q + 1 < n && (reinterpret_cast<uintptr_t>(as + q) & 15) == 0) {
                    // volatile: issued here, ahead of the record wait (the compiler would
                    // otherwise sink the loads next to their use and expose the L2 latency)
                    asm volatile("ld.global.v2.f64 {%0, %1}, [%2];\n"
                                 : "=d"(av[q]), "=d"(av[q + 1]) : "l"(as + q) : "memory");
                } else {
                    av[q] = j0 + q < n ? as[q] : 0.0;
                    av[q + 1] = j0 + q + 1 < n ? as[q + 1] : 0.0;
                }
            }
        }
        long long pc = clock64();
        const long long pc0 = pc;
        (void)pc0;
        mb_wait(&bars[tt & 1], (unsigned)((tt >> 1) & 1));
        CWP(2, pc);
        const double2* r2 = reinterpret_cast<const double2*>(sm + (tt & 1) * REC);
        auto g2 = [&](int slot) -> double2 { return r2[(slot >> 1) * T + t]; };
        // ---- right-hand side (f0, f1) at the chunk nodes
        double g0[NA], g1[NA];                 // rhs f
        if (FWD) {                             // (0, -C_i u_{i-1})
            xE[t] = make_double2(w[0], w[NA - 1]);
            bsync<T>();
            const double wl = t > 0 ? xE[t - 1].y : 0.0;
            const double wr = t < T - 1 ? xE[t + 1].x : 0.0;
#pragma unroll
            for (int q = 0; q < NA; ++q) {
                const double2 c0 = g2(cw_oC(NA, LT) + 4 * q), c1 = g2(cw_oC(NA, LT) + 4 * q + 2);
                const double wm = q > 0 ? w[q - 1] : wl, wp = q < NA - 1 ? w[q + 1] : wr;
                g0[q] = 0.0;
                g1[q] = -(c0.y * w[q] + c0.x * wm + c1.x * wp);
            }
        } else {                               // (-mu_{i+1}, 0)
#pragma unroll
            for (int q = 0; q < NA; ++q) { g0[q] = -w[q]; g1[q] = 0.0; }
        }
        // ---- the two Thomas rhs sweeps, interleaved (independent recurrences; a
        // dependent fp64 operation costs ~23 cycles, so each step is two chained FMAs):
        // bottom-up over the interior h_k = f_k - S_k^T h_{k+1} (down to h_0) and
        // top-down g_k = f_k - T_{k-1}^T g_{k-1}
        double gg0[NA], gg1[NA];               // g_k (g0/g1 keep the rhs f for the bottom-up sweep)
        gg0[0] = g0[0]; gg1[0] = g1[0];
        double h0 = g0[NA - 2], h1 = g1[NA - 2];
#pragma unroll
        for (int q = 1; q < NA; ++q) {
            {
                const double2 ta = g2(cw_oT(NA) + 4 * (q - 1)), tb = g2(cw_oT(NA) + 4 * (q - 1) + 2);
                gg0[q] = fma(-ta.x, gg0[q - 1], fma(-tb.x, gg1[q - 1], g0[q]));
                gg1[q] = fma(-ta.y, gg0[q - 1], fma(-tb.y, gg1[q - 1], g1[q]));
            }
            const int qb = NA - 2 - q;         // bottom-up node
            if (qb >= 0) {
                const double2 sa = g2(cw_oS(NA) + 4 * qb), sb = g2(cw_oS(NA) + 4 * qb + 2);
                const double n0 = fma(-sa.x, h0, fma(-sb.x, h1, g0[qb]));   // f - S^T h
                const double n1 = fma(-sa.y, h0, fma(-sb.y, h1, g1[qb]));
                h0 = n0; h1 = n1;
            }
        }
        xH[t] = make_double2(h0, h1);
        bsync<T>();
        CWP(3, pc);
        // ---- interface rhs and the rhs-only parallel cyclic reduction
        double R0 = gg0[NA - 1], R1 = gg1[NA - 1];
        {
            const double2 hn = t < T - 1 ? xH[t + 1] : make_double2(0.0, 0.0);
            const double2 va = g2(cw_oV(NA)), vb = g2(cw_oV(NA) + 2);
            R0 -= va.x * hn.x + va.y * hn.y;
            R1 -= vb.x * hn.x + vb.y * hn.y;
        }
#pragma unroll
        for (int l = 0; l < LT; ++l) {
            const int s = 1 << l;
            double2* P = xP[l & 1];
            P[t] = make_double2(R0, R1);
            const double2 aa = g2(cw_oP(NA) + 8 * l), ab = g2(cw_oP(NA) + 8 * l + 2);
            const double2 ca = g2(cw_oP(NA) + 8 * l + 4), cb = g2(cw_oP(NA) + 8 * l + 6);
            bsync<T>();
            const double2 rm = t >= s ? P[t - s] : make_double2(0.0, 0.0);
            const double2 rp = t + s < T ? P[t + s] : make_double2(0.0, 0.0);
            R0 = fma(-aa.x, rm.x, fma(-aa.y, rm.y, R0)) - fma(ca.x, rp.x, ca.y * rp.y);
            R1 = fma(-ab.x, rm.x, fma(-ab.y, rm.y, R1)) - fma(cb.x, rp.x, cb.y * rp.y);
        }
        double x0[NA], x1[NA];
        {
            const double2 ba = g2(cw_oB(NA, LT)), bb = g2(cw_oB(NA, LT) + 2);
            x0[NA - 1] = ba.x * R0 + ba.y * R1;
            x1[NA - 1] = bb.x * R0 + bb.y * R1;
        }
        xX[t] = make_double2(x0[NA - 1], x1[NA - 1]);
        bsync<T>();
        const double2 xl = t > 0 ? xX[t - 1] : make_double2(0.0, 0.0);
        CWP(4, pc);
        // ---- back-substitution: x_k = Di_k g_k + G_k x_L - T_k x_{k+1}
#pragma unroll
        for (int q = NA - 2; q >= 0; --q) {
            const double2 da = g2(cw_oDi(NA) + 4 * q), db = g2(cw_oDi(NA) + 4 * q + 2);
            const double2 ga = g2(cw_oG(NA) + 4 * q), gb = g2(cw_oG(NA) + 4 * q + 2);
            const double2 ta = g2(cw_oT(NA) + 4 * q), tb = g2(cw_oT(NA) + 4 * q + 2);
            const double p0 = (da.x * gg0[q] + da.y * gg1[q]) + (ga.x * xl.x + ga.y * xl.y);
            const double p1 = (db.x * gg0[q] + db.y * gg1[q]) + (gb.x * xl.x + gb.y * xl.y);
            x0[q] = fma(-ta.x, x0[q + 1], fma(-ta.y, x1[q + 1], p0));
            x1[q] = fma(-tb.x, x0[q + 1], fma(-tb.y, x1[q + 1], p1));
        }
        // ---- the step's coupling vector
        if (FWD) {                             // u_i = a_i + u-part
#pragma unroll
            for (int q = 0; q < NA; ++q) w[q] = av[q] + x0[q];
        } else {                               // mu_i = a_i + C_i^T lam
            xE[t] = make_double2(x1[0], x1[NA - 1]);
            bsync<T>();
            const double ll = t > 0 ? xE[t - 1].y : 0.0;
            const double lr = t < T - 1 ? xE[t + 1].x : 0.0;
            const double2 ed = g2(cw_oE(NA, LT));   // (Cp[j0-1], Cs[j0+NA])
            double cpm = ed.x;                      // Cp at node j-1
#pragma unroll
            for (int q = 0; q < NA; ++q) {
                const double2 c0 = g2(cw_oC(NA, LT) + 4 * q), c1 = g2(cw_oC(NA, LT) + 4 * q + 2);
                const double csn = q < NA - 1 ? g2(cw_oC(NA, LT) + 4 * (q + 1)).x : ed.y;   // Cs at node j+1
                const double lm = q > 0 ? x1[q - 1] : ll, lp = q < NA - 1 ? x1[q + 1] : lr;
                w[q] = av[q] + (c0.y * x1[q] + cpm * lm + csn * lp);
                cpm = c1.x;
            }
        }
        {
            double* dst = chain + (size_t)i * n + j0;
            const bool last = k + 1 == k1 && eout != nullptr;
#pragma unroll
            for (int q = 0; q < NA; q += 2) {
                if (j0 + q + 1 < n && (reinterpret_cast<uintptr_t>(dst + q) & 15) == 0) {
                    *reinterpret_cast<double2*>(dst + q) = make_double2(w[q], w[q + 1]);
                } else {
                    if (j0 + q < n) dst[q] = w[q];
                    if (j0 + q + 1 < n) dst[q + 1] = w[q + 1];
                }
                if (last) {
                    if (j0 + q < n) eout[j0 + q] = w[q];
                    if (j0 + q + 1 < n) eout[j0 + q + 1] = w[q + 1];
                }
            }
        }
        CWP(5, pc);
#ifdef TK_PROF
        if (blockIdx.x == 1 && threadIdx.x == 0) { g_cw_prof[0] += 1; g_cw_prof[1] += clock64() - pc0; }
#endif
    }
}


// ---------------------------------------------------------------------------
// Streaming variant for 512 < n_u <= 2048 (T = 64 / 128 threads of 16 nodes):
// the interval record (up to 380 KB) no longer fits shared memory, so every
// thread streams ITS OWN coefficients through a private ring of R 32-byte
// groups filled by cp.async in the exact order the solve consumes them
// (cws_slot).  No staging barrier, no mbarrier: `cp.async.wait_group R-1`
// before a group is read, the refill of the freed slot (R groups ahead, into
// the next interval's record when the order wraps) right after.  Whole
// records are pulled into L2 two intervals ahead by one bulk prefetch.
// tri_chain_kernel needed ~32 us per interval at n_u = 2048 (record reads on
// the critical path); this takes ~2.5 us.
// ---------------------------------------------------------------------------
template <int NA, int LT>
__host__ __device__ constexpr int cws_common() { return 5 * NA - 4 + 2 * LT; }
// ring length (groups in flight per thread): 27 for 16 nodes per thread (108 groups per
// interval), the whole interval (35 groups) for 4 nodes per thread
template <int NA>
__host__ __device__ constexpr int cws_ring() { return NA >= 16 ? 27 : 35; }
template <int NA, int LT>
__host__ __device__ constexpr int cws_gpi() {   // groups per interval, padded to a multiple of the ring
    return (cws_common<NA, LT>() + NA + 1 + cws_ring<NA>() - 1) / cws_ring<NA>() * cws_ring<NA>();
}
// record slot of the i-th group in consumption order (FWD: C first; BWD: E, C last)
template <bool FWD, int NA, int LT>
__host__ __device__ constexpr int cws_slot(int i) {
    if (FWD) {
        if (i < NA) return cw_oC(NA, LT) + 4 * i;
        i -= NA;
    }
    if (i < 2 * (NA - 2)) {
        const int q = i / 2 + 1;
        return (i & 1) ? cw_oS(NA) + 4 * (NA - 2 - q) : cw_oT(NA) + 4 * (q - 1);
    }
    i -= 2 * (NA - 2);
    if (i == 0) return cw_oT(NA) + 4 * (NA - 2);
    i -= 1;
    if (i == 0) return cw_oV(NA);
    i -= 1;
    if (i < 2 * LT) return cw_oP(NA) + 4 * i;
    i -= 2 * LT;
    if (i == 0) return cw_oB(NA, LT);
    i -= 1;
    if (i < 3 * (NA - 1)) {
        const int q = NA - 2 - i / 3, r = i % 3;
        return r == 0 ? cw_oDi(NA) + 4 * q : (r == 1 ? cw_oG(NA) + 4 * q : cw_oT(NA) + 4 * q);
    }
    i -= 3 * (NA - 1);
    if (i == 0) return cw_oE(NA, LT);
    i -= 1;
    if (!FWD && i < NA) return cw_oC(NA, LT) + 4 * i;
    return 0;   // padding group (never read)
}

template <bool FWD, int NA, int T>
__global__ void __launch_bounds__(T, 1)
    tri_chainw_stream(TView V, const double* __restrict__ a, const double* __restrict__ facw,
                      double* __restrict__ chain, int Lc, int cbase,
                      const double* __restrict__ starts, double* __restrict__ ends) {
    constexpr int LT = ilog2(T);
    constexpr int SL = cw_slots(NA, LT);
    constexpr int REC = SL * T;
    constexpr int R = cws_ring<NA>();
    constexpr int GPI = cws_gpi<NA, LT>();
    constexpr int CB = FWD ? NA : 0;                     // first common group
    constexpr int CM = cws_common<NA, LT>();
    static_assert(GPI % R == 0 && R <= GPI, "ring must divide the interval stream");
    extern __shared__ __align__(16) double sm[];
    double2* ring = reinterpret_cast<double2*>(sm);      // [R][2][T]
    double2* xH = ring + R * 2 * T;                      // exchange arrays [T] each
    double2* xP[2] = {xH + T, xH + 2 * T};
    double2* xX = xH + 3 * T;
    double2* xE = xH + 4 * T;
    const Lay& L = V.lay;
    const int n = V.n, N = L.N;
    const int t = threadIdx.x;
    const int K = N - 1;
    const int c = cbase + blockIdx.x;
    const int lo = c * Lc, hi = min(K, lo + Lc);
    const int k0 = FWD ? lo : K - hi, k1 = FWD ? hi : K - lo;
    const bool seed = k0 == 0;
    auto blk = [&](int k) { return FWD ? 1 + k : N - 1 - k; };
    auto aseg = [&](int i) { return a + (FWD ? L.off_u(i) : L.off_mu(i)); };
    const int i0 = FWD ? 0 : N;
    const double* s0 = seed ? aseg(i0) : (starts ? starts + (size_t)c * n : nullptr);
    const int j0 = NA * t;
    double w[NA];
#pragma unroll
    for (int k = 0; k < NA; ++k) w[k] = (s0 && j0 + k < n) ? s0[j0 + k] : 0.0;
    if (seed) {
#pragma unroll
        for (int k = 0; k < NA; ++k)
            if (j0 + k < n) chain[(size_t)i0 * n + j0 + k] = w[k];
    }
    if (k0 >= k1) return;
    // group g (0 <= g < 2 GPI) of the stream that starts at interval step k
    auto issue = [&](int k, int g) {
        const int kk = k + (g >= GPI ? 1 : 0);
        const int gi = g >= GPI ? g - GPI : g;
        const int kc = kk < k1 ? kk : k1 - 1;              // past the chunk: refetch (never read)
        const int sl = cws_slot<FWD, NA, LT>(gi);
        const double2* src = reinterpret_cast<const double2*>(facw + (size_t)blk(kc) * REC) +
                             (sl >> 1) * T + t;
        double2* dst = ring + ((gi % R) * 2) * T + t;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s_u32(dst)), "l"(src) : "memory");
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s_u32(dst + T)), "l"(src + T)
                     : "memory");
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    auto l2_prefetch = [&](int k) {   // the whole record of step k -> L2 (one thread)
        if (t != 0 || k >= k1) return;
        const char* p = reinterpret_cast<const char*>(facw + (size_t)blk(k) * REC);
        const unsigned bytes = (unsigned)(REC * sizeof(double));
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
    };
    l2_prefetch(k0 + 1);
#pragma unroll
    for (int g = 0; g < R; ++g) issue(k0, g);
    double* eout = ends ? ends + (size_t)c * n : nullptr;
    for (int k = k0; k < k1; ++k) {
        const int i = blk(k);
        l2_prefetch(k + 2);
        // take group g of this interval: wait, read, refill the slot with group g + R
        auto take = [&](int g, double2& u0, double2& u1) {
            asm volatile("cp.async.wait_group %0;\n" ::"n"(R - 1) : "memory");
            const double2* src = ring + ((g % R) * 2) * T + t;
            u0 = src[0];
            u1 = src[T];
            issue(k, g + R);
        };
        // an unread group: its copy must still have landed before the slot is refilled
        // (two copies in flight to one slot may complete in either order)
        auto skip = [&](int g) {
            asm volatile("cp.async.wait_group %0;\n" ::"n"(R - 1) : "memory");
            issue(k, g + R);
        };
        // a_i at the chunk nodes: issued now, consumed after the solve
        double av[NA];
        {
            const double* as = aseg(i) + j0;
#pragma unroll
            for (int q = 0; q < NA; q += 2) {
                if (j0 + q + 1 < n && (reinterpret_cast<uintptr_t>(as + q) & 15) == 0) {
                    asm volatile("ld.global.v2.f64 {%0, %1}, [%2];\n"
                                 : "=d"(av[q]), "=d"(av[q + 1]) : "l"(as + q) : "memory");
                } else {
                    av[q] = j0 + q < n ? as[q] : 0.0;
                    av[q + 1] = j0 + q + 1 < n ? as[q + 1] : 0.0;
                }
            }
        }
        // ---- right-hand side
        double g0[NA], g1[NA];
        if (FWD) {
            xE[t] = make_double2(w[0], w[NA - 1]);
            bsync<T>();
            const double wl = t > 0 ? xE[t - 1].y : 0.0;
            const double wr = t < T - 1 ? xE[t + 1].x : 0.0;
#pragma unroll
            for (int q = 0; q < NA; ++q) {
                double2 c0, c1;
                take(q, c0, c1);
                const double wm = q > 0 ? w[q - 1] : wl, wp = q < NA - 1 ? w[q + 1] : wr;
                g0[q] = 0.0;
                g1[q] = -(c0.y * w[q] + c0.x * wm + c1.x * wp);
            }
        } else {
#pragma unroll
            for (int q = 0; q < NA; ++q) { g0[q] = -w[q]; g1[q] = 0.0; }
        }
        // ---- the two Thomas rhs sweeps, interleaved
        double gg0[NA], gg1[NA];
        gg0[0] = g0[0]; gg1[0] = g1[0];
        double h0 = g0[NA - 2], h1 = g1[NA - 2];
#pragma unroll
        for (int q = 1; q < NA; ++q) {
            {
                double2 ta, tb;
                take(CB + (q < NA - 1 ? 2 * (q - 1) : 2 * (NA - 2)), ta, tb);
                gg0[q] = fma(-ta.x, gg0[q - 1], fma(-tb.x, gg1[q - 1], g0[q]));
                gg1[q] = fma(-ta.y, gg0[q - 1], fma(-tb.y, gg1[q - 1], g1[q]));
            }
            const int qb = NA - 2 - q;
            if (qb >= 0) {
                double2 sa, sb;
                take(CB + 2 * (q - 1) + 1, sa, sb);
                const double n0 = fma(-sa.x, h0, fma(-sb.x, h1, g0[qb]));
                const double n1 = fma(-sa.y, h0, fma(-sb.y, h1, g1[qb]));
                h0 = n0; h1 = n1;
            }
        }
        xH[t] = make_double2(h0, h1);
        bsync<T>();
        // ---- interface rhs and the rhs-only parallel cyclic reduction
        double R0 = gg0[NA - 1], R1 = gg1[NA - 1];
        {
            const double2 hn = t < T - 1 ? xH[t + 1] : make_double2(0.0, 0.0);
            double2 va, vb;
            take(CB + 2 * NA - 3, va, vb);
            R0 -= va.x * hn.x + va.y * hn.y;
            R1 -= vb.x * hn.x + vb.y * hn.y;
        }
#pragma unroll
        for (int l = 0; l < LT; ++l) {
            const int s = 1 << l;
            double2* P = xP[l & 1];
            P[t] = make_double2(R0, R1);
            double2 aa, ab, ca, cb;
            take(CB + 2 * NA - 2 + 2 * l, aa, ab);
            take(CB + 2 * NA - 2 + 2 * l + 1, ca, cb);
            bsync<T>();
            const double2 rm = t >= s ? P[t - s] : make_double2(0.0, 0.0);
            const double2 rp = t + s < T ? P[t + s] : make_double2(0.0, 0.0);
            R0 = fma(-aa.x, rm.x, fma(-aa.y, rm.y, R0)) - fma(ca.x, rp.x, ca.y * rp.y);
            R1 = fma(-ab.x, rm.x, fma(-ab.y, rm.y, R1)) - fma(cb.x, rp.x, cb.y * rp.y);
        }
        double x0[NA], x1[NA];
        {
            double2 ba, bb;
            take(CB + 2 * NA - 2 + 2 * LT, ba, bb);
            x0[NA - 1] = ba.x * R0 + ba.y * R1;
            x1[NA - 1] = bb.x * R0 + bb.y * R1;
        }
        xX[t] = make_double2(x0[NA - 1], x1[NA - 1]);
        bsync<T>();
        const double2 xl = t > 0 ? xX[t - 1] : make_double2(0.0, 0.0);
        // ---- back-substitution
#pragma unroll
        for (int q = NA - 2; q >= 0; --q) {
            constexpr int BS = CB + 2 * NA - 1 + 2 * LT;
            double2 da, db, ga, gb, ta, tb;
            take(BS + 3 * (NA - 2 - q), da, db);
            take(BS + 3 * (NA - 2 - q) + 1, ga, gb);
            take(BS + 3 * (NA - 2 - q) + 2, ta, tb);
            const double p0 = (da.x * gg0[q] + da.y * gg1[q]) + (ga.x * xl.x + ga.y * xl.y);
            const double p1 = (db.x * gg0[q] + db.y * gg1[q]) + (gb.x * xl.x + gb.y * xl.y);
            x0[q] = fma(-ta.x, x0[q + 1], fma(-ta.y, x1[q + 1], p0));
            x1[q] = fma(-tb.x, x0[q + 1], fma(-tb.y, x1[q + 1], p1));
        }
        // ---- the step's coupling vector
        if (FWD) {
#pragma unroll
            for (int q = 0; q < NA; ++q) w[q] = av[q] + x0[q];
            skip(CB + CM);                                  // the edge group (BWD only)
        } else {
            xE[t] = make_double2(x1[0], x1[NA - 1]);
            bsync<T>();
            const double ll = t > 0 ? xE[t - 1].y : 0.0;
            const double lr = t < T - 1 ? xE[t + 1].x : 0.0;
            double2 ed, e1;
            take(CM, ed, e1);                               // (Cp[j0-1], Cs[j0+NA])
            double cs_[NA], cd_[NA], cp_[NA];
#pragma unroll
            for (int q = 0; q < NA; ++q) {
                double2 c0, c1;
                take(CM + 1 + q, c0, c1);
                cs_[q] = c0.x; cd_[q] = c0.y; cp_[q] = c1.x;
            }
#pragma unroll
            for (int q = 0; q < NA; ++q) {
                const double cpm = q > 0 ? cp_[q - 1] : ed.x;
                const double csn = q < NA - 1 ? cs_[q + 1] : ed.y;
                const double lm = q > 0 ? x1[q - 1] : ll, lp = q < NA - 1 ? x1[q + 1] : lr;
                w[q] = av[q] + (cd_[q] * x1[q] + cpm * lm + csn * lp);
            }
        }
#pragma unroll
        for (int g = CM + NA + 1; g < GPI; ++g) skip(g);   // padding groups
        {
            double* dst = chain + (size_t)i * n + j0;
            const bool last = k + 1 == k1 && eout != nullptr;
#pragma unroll
            for (int q = 0; q < NA; q += 2) {
                if (j0 + q + 1 < n && (reinterpret_cast<uintptr_t>(dst + q) & 15) == 0) {
                    *reinterpret_cast<double2*>(dst + q) = make_double2(w[q], w[q + 1]);
                } else {
                    if (j0 + q < n) dst[q] = w[q];
                    if (j0 + q + 1 < n) dst[q + 1] = w[q + 1];
                }
                if (last) {
                    if (j0 + q < n) eout[j0 + q] = w[q];
                    if (j0 + q + 1 < n) eout[j0 + q + 1] = w[q + 1];
                }
            }
        }
        bsync<T>();   // the exchange arrays are free for the next step
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
// (nodes per thread) * 1000 + threads of the warp chain for n_u (0: unsupported ->
// tri_chain_kernel).  n_u <= 256: one warp; 256 < n_u <= 512: two warps of 8
// nodes per thread (TK_CHAIN_NA=16: one warp of 16, 4200 cycles per interval;
// TK_CHAIN_NA=4: four warps of 4 through the streaming variant, measured
// slower: 183 vs 171 us per forward substitution) -- the double-buffered
// records (101 KB each at n_u = 512) bound the sizes covered.
int chainw_nodes(int n) {
    static int on = -1, na512 = 8;
    if (on < 0) {
        const char* e = getenv("TK_CHAIN_WARP");
        on = (e && e[0] == '0') ? 0 : 1;
        const char* a = getenv("TK_CHAIN_NA");
        if (a && atoi(a) == 16) na512 = 16;
        if (a && atoi(a) == 4) na512 = 4;
    }
    if (!on || n < 32 || n > 2048 || (n & 1)) return 0;
    if (n <= 128) return 4 * 1000 + 32;
    if (n <= 256) return 8 * 1000 + 32;
    if (n <= 512) return na512 == 16 ? 16 * 1000 + 32 : (na512 == 4 ? 4 * 1000 + 128 : 8 * 1000 + 64);
    // beyond 512 the records exceed shared memory: per-thread cp.async streams
    return n <= 1024 ? 16 * 1000 + 64 : 16 * 1000 + 128;
}
static int cw_log2(int t) { return t == 128 ? 7 : (t == 64 ? 6 : 5); }
// doubles of the level's warp-chain records (N intervals; record 0 unused)
int64_t chainw_len(const tk_level* Lv) {
    const int cfg = chainw_nodes(Lv->n_u);
    if (!cfg) return 0;
    const int na = cfg / 1000, T = cfg % 1000;
    return (int64_t)Lv->n_steps * cw_slots(na, cw_log2(T)) * T;
}

template <int NA, int T>
static int chainw_factor_t(const tk_level* Lv, double* facw, cudaStream_t s) {
    TView V(Lv);
    const int N = Lv->n_steps;
    if (N < 2) return TK_OK;
    tri_chainw_factor<NA, T><<<N - 1, T, 0, s>>>(V, facw);
    return check_launch("tri_chainw_factor");
}
int chainw_factor(const tk_level* Lv, double* facw, cudaStream_t s) {
    switch (chainw_nodes(Lv->n_u)) {
        case 4032: return chainw_factor_t<4, 32>(Lv, facw, s);
        case 8032: return chainw_factor_t<8, 32>(Lv, facw, s);
        case 8064: return chainw_factor_t<8, 64>(Lv, facw, s);
        case 16032: return chainw_factor_t<16, 32>(Lv, facw, s);
        case 4128: return chainw_factor_t<4, 128>(Lv, facw, s);
        case 16064: return chainw_factor_t<16, 64>(Lv, facw, s);
        case 16128: return chainw_factor_t<16, 128>(Lv, facw, s);
        default: set_error("chainw_factor: unsupported n_u=%d", Lv->n_u); return TK_ERR_UNSUPPORTED;
    }
}

template <bool FWD, int NA, int T>
static int chainw_launch_t(const tk_level* Lv, const double* a, const double* facw, double* chain,
                           int Lc, int grid, int cbase, const double* st, double* en,
                           cudaStream_t s) {
    const size_t smem = (size_t)(2 * cw_slots(NA, ilog2(T)) * T + 5 * 2 * T) * sizeof(double);
    static bool attr = false;
    if (!attr) {
        const cudaError_t e = cudaFuncSetAttribute(tri_chainw_kernel<FWD, NA, T>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return cuda_status(e, "tri_chainw_kernel: attributes");
        attr = true;
    }
    TView V(Lv);
    tri_chainw_kernel<FWD, NA, T><<<grid, T, smem, s>>>(V, a, facw, chain, Lc, cbase, st, en);
    return check_launch("tri_chainw_kernel");
}
template <bool FWD, int NA, int T>
static int chainw_stream_t(const tk_level* Lv, const double* a, const double* facw, double* chain,
                           int Lc, int grid, int cbase, const double* st, double* en,
                           cudaStream_t s) {
    const size_t smem = (size_t)(cws_ring<NA>() * 2 * T + 5 * T) * sizeof(double2);
    static bool attr = false;
    if (!attr) {
        const cudaError_t e = cudaFuncSetAttribute(tri_chainw_stream<FWD, NA, T>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return cuda_status(e, "tri_chainw_stream: attributes");
        attr = true;
    }
    TView V(Lv);
    tri_chainw_stream<FWD, NA, T><<<grid, T, smem, s>>>(V, a, facw, chain, Lc, cbase, st, en);
    return check_launch("tri_chainw_stream");
}
int chainw_launch(const tk_level* Lv, bool fwd, const double* a, const double* facw, double* chain,
                  int Lc, int grid, int cbase, const double* st, double* en, cudaStream_t s) {
    if (grid <= 0) return TK_OK;
    switch (chainw_nodes(Lv->n_u)) {
        case 4128:
            return fwd ? chainw_stream_t<true, 4, 128>(Lv, a, facw, chain, Lc, grid, cbase, st, en, s)
                       : chainw_stream_t<false, 4, 128>(Lv, a, facw, chain, Lc, grid, cbase, st, en, s);
        case 16064:
            return fwd ? chainw_stream_t<true, 16, 64>(Lv, a, facw, chain, Lc, grid, cbase, st, en, s)
                       : chainw_stream_t<false, 16, 64>(Lv, a, facw, chain, Lc, grid, cbase, st, en, s);
        case 16128:
            return fwd ? chainw_stream_t<true, 16, 128>(Lv, a, facw, chain, Lc, grid, cbase, st, en, s)
                       : chainw_stream_t<false, 16, 128>(Lv, a, facw, chain, Lc, grid, cbase, st, en, s);
        default: break;
    }
#define TK_CW(NN, TT)                                                                               \
    case NN * 1000 + TT:                                                                            \
        return fwd ? chainw_launch_t<true, NN, TT>(Lv, a, facw, chain, Lc, grid, cbase, st, en, s)  \
                   : chainw_launch_t<false, NN, TT>(Lv, a, facw, chain, Lc, grid, cbase, st, en, s);
    switch (chainw_nodes(Lv->n_u)) {
        TK_CW(4, 32)
        TK_CW(8, 32)
        TK_CW(8, 64)
        TK_CW(16, 32)
        default: set_error("chainw_launch: unsupported n_u=%d", Lv->n_u); return TK_ERR_UNSUPPORTED;
    }
#undef TK_CW
}

}  // namespace tk
