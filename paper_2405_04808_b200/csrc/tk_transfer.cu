// Time-level transfers on the reference layout (multigrid.py:95-132):
// states/multipliers (u, v, lam, mu) use injection down / linear interpolation
// up; piecewise-constant controls use 2-interval averages down / copies up.
//
// The kernels run over a time slab of FINE block rows [r0, r1) (the whole
// level is the slab [0, N+1)).  Restriction: one thread per element of the
// output slice, whose global offset gives (block row, variable kind,
// component, time index).  Prolongation and the restricted residual after a
// zero-start sweep: one CTA per block row (n_u >= 32, 16-byte streams) or
// one thread per block row (tiny rows); every segment of a row is one kind at
// one time, so its sources are located once.  Restriction is slab-local;
// prolongation reads two halo segments: the previous slab's last coarse
// (u, lam) and the next slab's first coarse (v, mu).
#include "tk_common.cuh"

namespace tk {

enum Kind { KU = 0, KV = 1, KZ = 2, KM = 3, KL = 4 };

// Decode a global offset g of layout L into (kind, component, time index t).
__device__ __forceinline__ void decode(const Lay& L, int64_t g, int& kind, int& c, int& t) {
    const int nu = L.nu, nz = L.nz;
    if (g < L.F) {                               // block 0: u1 z1 lam1
        const int o = (int)g;
        t = 1;
        if (o < nu) { kind = KU; c = o; }
        else if (o < nu + nz) { kind = KZ; c = o - nu; }
        else { kind = KL; c = o - nu - nz; }
        return;
    }
    const int64_t q = g - L.F;
    int i = (int)(q / L.m) + 1;
    int o = (int)(q - (int64_t)(i - 1) * L.m);
    if (i >= L.N) {                              // last block: v_N mu_N
        i = L.N;
        o = (int)(g - L.start(L.N));
        t = L.N;
        if (o < nu) { kind = KV; c = o; } else { kind = KM; c = o - nu; }
        return;
    }
    // interior block i: v_i u_{i+1} z_{i+1} mu_i lam_{i+1}
    if (o < nu) { kind = KV; c = o; t = i; }
    else if (o < 2 * nu) { kind = KU; c = o - nu; t = i + 1; }
    else if (o < 2 * nu + nz) { kind = KZ; c = o - 2 * nu; t = i + 1; }
    else if (o < 3 * nu + nz) { kind = KM; c = o - 2 * nu - nz; t = i; }
    else { kind = KL; c = o - 3 * nu - nz; t = i + 1; }
}

__device__ __forceinline__ int64_t kind_off(const Lay& L, int kind, int t) {
    switch (kind) {
        case KU: return L.t_u(t);
        case KV: return L.t_v(t);
        case KZ: return L.t_z(t);
        case KM: return L.t_mu(t);
        default: return L.t_l(t);
    }
}


__global__ void restrict_kernel(Lay Lf, Lay Lc, int64_t fbase, int64_t cbase, int64_t clen,
                                const double* __restrict__ xf, double* __restrict__ xc) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < clen;
         k += (int64_t)gridDim.x * blockDim.x) {
        int kind, c, t;
        decode(Lc, cbase + k, kind, c, t);
        if (kind == KZ) {
            const double a = xf[kind_off(Lf, KZ, 2 * t - 1) + c - fbase];
            const double b = xf[kind_off(Lf, KZ, 2 * t) + c - fbase];
            xc[k] = 0.5 * (a + b);
        } else {
            xc[k] = xf[kind_off(Lf, kind, 2 * t) + c - fbase];
        }
    }
}


// Row-based prolong-add: one CTA per fine block row; every segment of the row
// is one kind at one fine time, so its (at most two) coarse source segments
// are located once per CTA and the row is streamed with 16-byte accesses
// when the layout allows.
__device__ __forceinline__ const double* coarse_seg(const Lay& Lc, const double* xc, int64_t cbase,
                                                    int64_t clen, const double* hprev,
                                                    const double* hnext, int kind, int t) {
    const int64_t g = kind_off(Lc, kind, t);
    const int64_t l = g - cbase;
    if (l >= 0 && l < clen) return xc + l;
    if (l < 0) return hprev + (kind == KU ? 0 : Lc.nu);   // previous slab: (u, lam)
    return hnext + (kind == KV ? 0 : Lc.nu);                // next slab: (v, mu)
}

__global__ void __launch_bounds__(256) prolong_rows_kernel(Lay Lf, Lay Lc, int64_t fbase, int r0,
                                                           int r1, int64_t cbase, int64_t clen,
                                                           const double* __restrict__ xc,
                                                           const double* __restrict__ hprev,
                                                           const double* __restrict__ hnext,
                                                           double* __restrict__ xf, bool vec) {
    for (int i = r0 + blockIdx.x; i < r1; i += gridDim.x) {
        // segments of row i: kind, fine time, offset
        int kinds[5], ts[5];
        int64_t offs[5];
        int ns = 0;
        auto add = [&](int k, int t, int64_t o) { kinds[ns] = k; ts[ns] = t; offs[ns] = o; ++ns; };
        if (i >= 1) add(KV, i, Lf.off_v(i));
        if (i < Lf.N) { add(KU, i + 1, Lf.off_u(i)); add(KZ, i + 1, Lf.off_z(i)); }
        if (i >= 1) add(KM, i, Lf.off_mu(i));
        if (i < Lf.N) add(KL, i + 1, Lf.off_l(i));
        if (vec && Lf.nu <= 2 * (int)blockDim.x && Lf.nz <= 2 * (int)blockDim.x) {
            // one double2 per thread and segment: every load of the row is issued
            // before the first store (the stores could alias later loads)
            constexpr int qk[5] = {KV, KU, KZ, KM, KL};
            double2 d[5], u[5], w[5];
            double* dsts[5];
            bool on[5], two[5];
            const int k = 2 * threadIdx.x;
#pragma unroll
            for (int q = 0; q < 5; ++q) {
                const int kind = qk[q];
                const bool vm = kind == KV || kind == KM;
                const int t = vm ? i : i + 1;
                on[q] = (vm ? i >= 1 : i < Lf.N) && k < (kind == KZ ? Lf.nz : Lf.nu);
                two[q] = false;
                dsts[q] = xf;
                if (!on[q]) continue;
                const int64_t off = kind == KV ? Lf.off_v(i) : kind == KU ? Lf.off_u(i) :
                                    kind == KZ ? Lf.off_z(i) : kind == KM ? Lf.off_mu(i) : Lf.off_l(i);
                dsts[q] = xf + (off - fbase) + k;
                const double* a;
                const double* b = nullptr;
                if (kind == KZ) {
                    a = coarse_seg(Lc, xc, cbase, clen, hprev, hnext, KZ, (t + 1) / 2);
                } else if ((t & 1) == 0) {
                    a = coarse_seg(Lc, xc, cbase, clen, hprev, hnext, kind, t / 2);
                } else if (t == 1) {
                    a = coarse_seg(Lc, xc, cbase, clen, hprev, hnext, kind, 1);
                } else {
                    a = coarse_seg(Lc, xc, cbase, clen, hprev, hnext, kind, (t - 1) / 2);
                    b = coarse_seg(Lc, xc, cbase, clen, hprev, hnext, kind, (t + 1) / 2);
                }
                two[q] = b != nullptr;
                d[q] = *reinterpret_cast<const double2*>(dsts[q]);
                u[q] = *reinterpret_cast<const double2*>(a + k);
                if (b) w[q] = *reinterpret_cast<const double2*>(b + k);
            }
#pragma unroll
            for (int q = 0; q < 5; ++q) {
                if (!on[q]) continue;
                double2 o = d[q];
                if (two[q]) {
                    o.x = o.x + 0.5 * (u[q].x + w[q].x);
                    o.y = o.y + 0.5 * (u[q].y + w[q].y);
                } else {
                    o.x = o.x + u[q].x;
                    o.y = o.y + u[q].y;
                }
                *reinterpret_cast<double2*>(dsts[q]) = o;
            }
            continue;
        }
        for (int q = 0; q < ns; ++q) {
            const int kind = kinds[q], t = ts[q];
            const int len = kind == KZ ? Lf.nz : Lf.nu;
            double* dst = xf + (offs[q] - fbase);
            const double* a;
            const double* b = nullptr;
            if (kind == KZ) {
                a = coarse_seg(Lc, xc, cbase, clen, hprev, hnext, KZ, (t + 1) / 2);
            } else if ((t & 1) == 0) {
                a = coarse_seg(Lc, xc, cbase, clen, hprev, hnext, kind, t / 2);
            } else if (t == 1) {
                a = coarse_seg(Lc, xc, cbase, clen, hprev, hnext, kind, 1);
            } else {
                a = coarse_seg(Lc, xc, cbase, clen, hprev, hnext, kind, (t - 1) / 2);
                b = coarse_seg(Lc, xc, cbase, clen, hprev, hnext, kind, (t + 1) / 2);
            }
            if (vec) {   // every segment 16-byte aligned, len even
                const int h = len / 2;
                for (int k = threadIdx.x; k < h; k += blockDim.x) {
                    double2 d = reinterpret_cast<double2*>(dst)[k];
                    const double2 u = reinterpret_cast<const double2*>(a)[k];
                    if (b) {
                        const double2 w = reinterpret_cast<const double2*>(b)[k];
                        d.x = d.x + 0.5 * (u.x + w.x);
                        d.y = d.y + 0.5 * (u.y + w.y);
                    } else {
                        d.x = d.x + u.x;
                        d.y = d.y + u.y;
                    }
                    reinterpret_cast<double2*>(dst)[k] = d;
                }
            } else {
                for (int k = threadIdx.x; k < len; k += blockDim.x)
                    dst[k] = dst[k] + (b ? 0.5 * (a[k] + b[k]) : a[k]);
            }
        }
    }
}

// Tiny rows (van der Pol, n_u < 32): one THREAD per fine block row (the
// element-wise kernel spent its time in the 64-bit index decode); same
// arithmetic as prolong_rows_kernel's scalar path.
__global__ void prolong_small_kernel(Lay Lf, Lay Lc, int64_t fbase, int r0, int r1, int64_t cbase,
                                     int64_t clen, const double* __restrict__ xc,
                                     const double* __restrict__ hprev,
                                     const double* __restrict__ hnext, double* __restrict__ xf) {
    // a CTA owns blockDim.x consecutive fine rows: their contiguous slice of xf
    // is staged through shared memory with coalesced loads/stores, and each
    // thread updates its own row there
    extern __shared__ double sx[];
    const int rb = blockDim.x;
    for (int i0 = r0 + blockIdx.x * rb; i0 < r1; i0 += gridDim.x * rb) {
        const int i1 = min(i0 + rb, r1);
        const int64_t g0 = Lf.start(i0), g1 = (i1 == Lf.N + 1) ? Lf.dim() : Lf.start(i1);
        const int len = (int)(g1 - g0);
        double* row0 = xf + (g0 - fbase);
        for (int k = threadIdx.x; k < len; k += rb) sx[k] = row0[k];
        __syncthreads();
        const int i = i0 + threadIdx.x;
        if (i < i1) {
            auto seg = [&](int kind, int t, int64_t off, int ln) {
                double* dst = sx + (off - g0);
                const double* a;
                const double* b = nullptr;
                if (kind == KZ) {
                    a = coarse_seg(Lc, xc, cbase, clen, hprev, hnext, KZ, (t + 1) / 2);
                } else if ((t & 1) == 0) {
                    a = coarse_seg(Lc, xc, cbase, clen, hprev, hnext, kind, t / 2);
                } else if (t == 1) {
                    a = coarse_seg(Lc, xc, cbase, clen, hprev, hnext, kind, 1);
                } else {
                    a = coarse_seg(Lc, xc, cbase, clen, hprev, hnext, kind, (t - 1) / 2);
                    b = coarse_seg(Lc, xc, cbase, clen, hprev, hnext, kind, (t + 1) / 2);
                }
                for (int k = 0; k < ln; ++k) {
                    const double val = b ? 0.5 * (a[k] + b[k]) : a[k];
                    dst[k] = dst[k] + val;
                }
            };
            if (i >= 1) seg(KV, i, Lf.off_v(i), Lf.nu);
            if (i < Lf.N) {
                seg(KU, i + 1, Lf.off_u(i), Lf.nu);
                seg(KZ, i + 1, Lf.off_z(i), Lf.nz);
            }
            if (i >= 1) seg(KM, i, Lf.off_mu(i), Lf.nu);
            if (i < Lf.N) seg(KL, i + 1, Lf.off_l(i), Lf.nu);
        }
        __syncthreads();
        for (int k = threadIdx.x; k < len; k += rb) row0[k] = sx[k];
        __syncthreads();
    }
}

// rc = R (b - A x) for x = ONE block-Jacobi sweep from zero, x = omega D^{-1} b
// (the pre-smoothing of every V-cycle level, multigrid.py:284-288).  Then
// D x = omega b, so  b - A x = (1 - omega) b - (L + U) x: the only other
// terms are the continuity couplings, r_mu(t) -= u_t and r_u(t) -= mu_t
// (kkt.py:6-16).  Injection keeps fine time 2T for u, v, lam, mu and averages
// z over 2T-1, 2T.  One thread per coarse element; b is not read when omega
// == 1, and x only at the u and mu segments the coarse rows inject.
static void slab_geom(const Lay& Lf, const Lay& Lc, int r0, int r1, int64_t& fbase,
                      int64_t& flen, int64_t& cbase, int64_t& clen);

// Time slab of fine rows [r0, r1): the coupling partners outside the slab are
// the halo segments (u of row r0-1 = u_{r0}, mu of row r1 = mu_{r1}).
// Row-based variant: one CTA per coarse block row; each of its segments is one
// (kind, coarse time) whose sources are located once, then streamed (16-byte
// accesses when aligned).  With
// omega == 1 the v, z, lam segments are zero and u, mu the negated couplings.
__global__ void __launch_bounds__(256) restrict_jacobi0_rows(Lay Lf, Lay Lc, int64_t fbase, int64_t cbase,
                                                             int c0, int c1, int r0, int r1,
                                                             const double* __restrict__ b,
                                                             const double* __restrict__ x,
                                                             const double* __restrict__ hu,
                                                             const double* __restrict__ hm, double omega,
                                                             double* __restrict__ rc, bool vec) {
    const double c1w = 1.0 - omega;
    for (int c = c0 + blockIdx.x; c < c1; c += gridDim.x) {
        int kinds[5], ts[5];
        int64_t offs[5];
        int ns = 0;
        auto add = [&](int k, int t, int64_t o) { kinds[ns] = k; ts[ns] = t; offs[ns] = o; ++ns; };
        if (c >= 1) add(KV, c, Lc.off_v(c));
        if (c < Lc.N) { add(KU, c + 1, Lc.off_u(c)); add(KZ, c + 1, Lc.off_z(c)); }
        if (c >= 1) add(KM, c, Lc.off_mu(c));
        if (c < Lc.N) add(KL, c + 1, Lc.off_l(c));
        for (int q = 0; q < ns; ++q) {
            const int kind = kinds[q], t = ts[q], ft = 2 * t;
            const int len = kind == KZ ? Lf.nz : Lf.nu;
            double* dst = rc + (offs[q] - cbase);
            const double* b1 = nullptr;   // c1w * b (z: average of fine 2t-1, 2t)
            const double* b2 = nullptr;
            if (c1w != 0.0) {
                if (kind == KZ) {
                    b1 = b + (kind_off(Lf, KZ, ft - 1) - fbase);
                    b2 = b + (kind_off(Lf, KZ, ft) - fbase);
                } else {
                    b1 = b + (kind_off(Lf, kind, ft) - fbase);
                }
            }
            const double* xs = nullptr;   // the continuity coupling
            if (kind == KM) xs = (ft - 1 >= r0) ? x + (kind_off(Lf, KU, ft) - fbase) : hu;
            else if (kind == KU) xs = (ft < r1) ? x + (kind_off(Lf, KM, ft) - fbase) : hm;
            auto val = [&](int k) -> double {
                double v = b1 == nullptr ? 0.0 : (b2 ? c1w * (0.5 * (b1[k] + b2[k])) : c1w * b1[k]);
                if (xs) v -= xs[k];
                return v;
            };
            if (vec) {
                for (int k = 2 * threadIdx.x; k < len; k += 2 * blockDim.x) {
                    double2 o;
                    if (b1 == nullptr && xs) {
                        const double2 u = *reinterpret_cast<const double2*>(xs + k);
                        o.x = 0.0 - u.x;
                        o.y = 0.0 - u.y;
                    } else {
                        o.x = val(k);
                        o.y = val(k + 1);
                    }
                    *reinterpret_cast<double2*>(dst + k) = o;
                }
            } else {
                for (int k = threadIdx.x; k < len; k += blockDim.x) dst[k] = val(k);
            }
        }
    }
}

// Tiny rows: one THREAD per coarse block row, same arithmetic as the kernels above.
__global__ void restrict_jacobi0_small(Lay Lf, Lay Lc, int64_t fbase, int64_t cbase, int c0, int c1,
                                       int r0, int r1, const double* __restrict__ b,
                                       const double* __restrict__ x, const double* __restrict__ hu,
                                       const double* __restrict__ hm, double omega,
                                       double* __restrict__ rc) {
    // a CTA owns blockDim.x consecutive coarse rows; each thread writes its row
    // into shared memory, the contiguous slice leaves with coalesced stores
    extern __shared__ double sx[];
    const double c1w = 1.0 - omega;
    const int rb = blockDim.x;
    for (int q0 = c0 + blockIdx.x * rb; q0 < c1; q0 += gridDim.x * rb) {
        const int q1 = min(q0 + rb, c1);
        const int64_t g0 = Lc.start(q0), g1 = (q1 == Lc.N + 1) ? Lc.dim() : Lc.start(q1);
        const int len = (int)(g1 - g0);
        const int c = q0 + threadIdx.x;
        if (c < q1) {
            auto seg = [&](int kind, int t, int64_t off, int ln) {
                const int ft = 2 * t;
                double* dst = sx + (off - g0);
                const double* xs = nullptr;
                if (kind == KM) xs = (ft - 1 >= r0) ? x + (kind_off(Lf, KU, ft) - fbase) : hu;
                else if (kind == KU) xs = (ft < r1) ? x + (kind_off(Lf, KM, ft) - fbase) : hm;
                for (int k = 0; k < ln; ++k) {
                    double v;
                    if (kind == KZ)
                        v = c1w == 0.0 ? 0.0
                                       : c1w * (0.5 * (b[kind_off(Lf, KZ, ft - 1) + k - fbase] +
                                                        b[kind_off(Lf, KZ, ft) + k - fbase]));
                    else
                        v = c1w == 0.0 ? 0.0 : c1w * b[kind_off(Lf, kind, ft) + k - fbase];
                    if (xs) v -= xs[k];
                    dst[k] = v;
                }
            };
            if (c >= 1) seg(KV, c, Lc.off_v(c), Lc.nu);
            if (c < Lc.N) {
                seg(KU, c + 1, Lc.off_u(c), Lc.nu);
                seg(KZ, c + 1, Lc.off_z(c), Lc.nz);
            }
            if (c >= 1) seg(KM, c, Lc.off_mu(c), Lc.nu);
            if (c < Lc.N) seg(KL, c + 1, Lc.off_l(c), Lc.nu);
        }
        __syncthreads();
        double* out = rc + (g0 - cbase);
        for (int k = threadIdx.x; k < len; k += rb) out[k] = sx[k];
        __syncthreads();
    }
}

// rows per CTA of the tiny-row kernels: a power of two, <= 256, with the
// CTA's rows (rb * m doubles) within 48 KB of shared memory
static int small_rows_per_cta(int m) {
    int rb = 256;
    while (rb > 32 && (int64_t)rb * m * 8 > 48 * 1024) rb >>= 1;
    return rb;
}

int restrict_jacobi0_launch(int n_fine, int nu, int nz, int r0, int r1, const double* b,
                            const double* x, const double* hu, const double* hm, double omega,
                            double* rc, cudaStream_t s) {
    Lay Lf(n_fine, nu, nz), Lc(n_fine / 2, nu, nz);
    if (r1 <= 0) r1 = n_fine + 1;
    if (r0 < 0 || r0 >= r1 || r1 > n_fine + 1 || (r0 & 1) || ((r1 & 1) && r1 != n_fine + 1)) {
        set_error("restrict_jacobi0: bad fine slab [%d, %d) for N=%d (edges must be even)", r0, r1,
                  n_fine);
        return TK_ERR_ARG;
    }
    if ((r0 > 0 && !hu) || (r1 <= n_fine && !hm)) {
        set_error("restrict_jacobi0: slab [%d, %d) needs its halo segments", r0, r1);
        return TK_ERR_ARG;
    }
    int64_t fbase, flen, cbase, clen;
    slab_geom(Lf, Lc, r0, r1, fbase, flen, cbase, clen);
    if (nu >= 32) {   // row-based (the element-wise kernel for tiny rows)
        const int c0 = r0 / 2, c1 = (r1 == n_fine + 1) ? Lc.N + 1 : r1 / 2;
        auto al = [](const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
        const bool vec = (nu % 2 == 0) && (nz % 2 == 0) && (fbase % 2 == 0) && (cbase % 2 == 0) &&
                         al(b) && al(x) && al(hu) && al(hm) && al(rc);
        const int rows = c1 - c0;
        restrict_jacobi0_rows<<<rows, nu >= 512 ? 256 : 128, 0, s>>>(Lf, Lc, fbase, cbase, c0, c1, r0, r1, b,
                                                                    x, hu, hm, omega, rc, vec);
        return check_launch("restrict_jacobi0_rows");
    }
    {   // tiny rows: one thread per coarse block row
        const int c0 = r0 / 2, c1 = (r1 == n_fine + 1) ? Lc.N + 1 : r1 / 2;
        const int rows = c1 - c0;
        const int rb = small_rows_per_cta(Lc.m);
        restrict_jacobi0_small<<<grid_for(rows, rb, 148 * 8), rb, (size_t)rb * Lc.m * 8, s>>>(
            Lf, Lc, fbase, cbase, c0, c1, r0, r1, b, x, hu, hm, omega, rc);
        return check_launch("restrict_jacobi0_small");
    }
}

// fine rows [r0, r1) -> coarse rows [r0/2, r1/2) (through N/2 for the last slab)
static void slab_geom(const Lay& Lf, const Lay& Lc, int r0, int r1, int64_t& fbase,
                      int64_t& flen, int64_t& cbase, int64_t& clen) {
    const int c0 = r0 / 2;
    const int c1 = (r1 == Lf.N + 1) ? Lc.N + 1 : r1 / 2;
    fbase = Lf.start(r0);
    flen = (r1 == Lf.N + 1 ? Lf.dim() : Lf.start(r1)) - fbase;
    cbase = Lc.start(c0);
    clen = (c1 == Lc.N + 1 ? Lc.dim() : Lc.start(c1)) - cbase;
}

int transfer_launch(int restrict_op, int n_fine, int nu, int nz, int r0, int r1, const double* in,
                    const double* hprev, const double* hnext, double* out, cudaStream_t s) {
    Lay Lf(n_fine, nu, nz), Lc(n_fine / 2, nu, nz);
    if (r1 <= 0) r1 = n_fine + 1;
    if (r0 < 0 || r0 >= r1 || r1 > n_fine + 1 || (r0 & 1) || ((r1 & 1) && r1 != n_fine + 1)) {
        set_error("transfer: bad fine slab [%d, %d) for N=%d (edges must be even)", r0, r1,
                  n_fine);
        return TK_ERR_ARG;
    }
    int64_t fbase, flen, cbase, clen;
    slab_geom(Lf, Lc, r0, r1, fbase, flen, cbase, clen);
    const bool need_prev = r0 > 0, need_next = r1 <= n_fine;
    const int th = 256;
    if (restrict_op) {
        restrict_kernel<<<grid_for(clen, th, 148 * 32), th, 0, s>>>(Lf, Lc, fbase, cbase, clen,
                                                                    in, out);
    } else {
        if ((need_prev && !hprev) || (need_next && !hnext)) {
            set_error("prolong_add: slab [%d, %d) needs its coarse halo segments", r0, r1);
            return TK_ERR_ARG;
        }
        auto al = [](const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
        const bool vec = (nu % 2 == 0) && (nz % 2 == 0) && (fbase % 2 == 0) && (cbase % 2 == 0) &&
                         al(in) && al(out) && al(hprev) && al(hnext);
        if (nu < 32) {   // tiny rows (van der Pol): one thread per fine block row
            const int rows = r1 - r0;
            const int rb = small_rows_per_cta((int)Lf.m);
            prolong_small_kernel<<<grid_for(rows, rb, 148 * 8), rb, (size_t)rb * Lf.m * 8, s>>>(
                Lf, Lc, fbase, r0, r1, cbase, clen, in, hprev, hnext, out);
            return check_launch("transfer");
        }
        const int rows = r1 - r0;
        const int pth = nu >= 512 ? 256 : 128;
        prolong_rows_kernel<<<rows < (1 << 30) ? rows : (1 << 30), pth, 0, s>>>(
            Lf, Lc, fbase, r0, r1, cbase, clen, in, hprev, hnext, out, vec);
    }
    return check_launch("transfer");
}

}  // namespace tk
