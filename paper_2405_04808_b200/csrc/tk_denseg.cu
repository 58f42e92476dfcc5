// DENSE family, general sizes: stage blocks K_i, C_i (n_u x n_u), B_i
// (n_u x n_z) and weights stored dense, for 4 < n_u <= 40 or 4 < n_z <= 8 --
// what the reference's DiagonalSolver handles for any ProblemSpec
// (kkt.py:279-389; e.g. its heat-Neumann problem, problems.py:218-266:
// n_z = 1 boundary control, n_u = n_cells + 1).  The register kernels of
// tk_dense.cu are templated on n_u, n_z <= 4; here one WARP owns a block row,
// its vectors and the local saddle system live in shared memory:
//
//   v = -r_mu;  [Qu 0 K^T; 0 Qz B^T; K B 0] (u, z, lam) = (r_u, r_z, r_lam - C v)
//   by Gaussian elimination with partial pivoting;  mu = Qv v + C^T lam - r_v,
//
// the exact D_i^{-1} of DiagonalSolver.solve_all without forming the
// (4n_u+n_z)^2 inverse.  Same data layout as the small DENSE family
// (tk_level: K, C [N][nu][nu], B [N][nu][nz], Qm, Ql [nu][nu], Qz [nz][nz]).
// Throughput is not the point of this family (desk-size generic problems).
#include "tk_common.cuh"

namespace tk {

namespace {

struct GView {
    Lay lay;
    Slab sl;
    const double *K, *C, *B, *Qm, *Ql, *Qz;
    int nu, nz;
    GView(const tk_level* L)
        : lay(L->n_steps, L->n_u, L->n_z), sl(L, Lay(L->n_steps, L->n_u, L->n_z)), K(L->K),
          C(L->C), B(L->B), Qm(L->Qm), Ql(L->Ql), Qz(L->Qz), nu(L->n_u), nz(L->n_z) {}
    __device__ const double* Ki(int i) const { return K + (size_t)(i - sl.r0) * nu * nu; }
    __device__ const double* Ci(int i) const { return C + (size_t)(i - sl.r0) * nu * nu; }
    __device__ const double* Bi(int i) const { return B + (size_t)(i - sl.r0) * nu * nz; }
};

enum GMode { G_APPLY = 0, G_APPLY_DIAG = 1, G_RESIDUAL = 2, G_SOLVE = 3, G_JACOBI = 4 };

// local row vector: [v(nu) u(nu) z(nz) m(nu) l(nu)]
struct Off {
    int v, u, z, m, l, len;
    __device__ Off(int nu, int nz) : v(0), u(nu), z(2 * nu), m(2 * nu + nz), l(3 * nu + nz), len(4 * nu + nz) {}
};

__device__ void load_row(const GView& V, int i, const double* x, double* s) {
    const Lay& L = V.lay;
    const Off o(V.nu, V.nz);
    const int lane = threadIdx.x & 31;
    for (int e = lane; e < o.len; e += 32) s[e] = 0.0;
    __syncwarp();
    if (!x) return;
    const int64_t bs = V.sl.base;
    if (i >= 1) {
        const double* pv = x + (L.off_v(i) - bs);
        const double* pm = x + (L.off_mu(i) - bs);
        for (int e = lane; e < V.nu; e += 32) { s[o.v + e] = pv[e]; s[o.m + e] = pm[e]; }
    }
    if (i < L.N) {
        const double* pu = x + (L.off_u(i) - bs);
        const double* pz = x + (L.off_z(i) - bs);
        const double* pl = x + (L.off_l(i) - bs);
        for (int e = lane; e < V.nu; e += 32) { s[o.u + e] = pu[e]; s[o.l + e] = pl[e]; }
        for (int e = lane; e < V.nz; e += 32) s[o.z + e] = pz[e];
    }
    __syncwarp();
}

__device__ void store_row(const GView& V, int i, double* y, const double* s) {
    const Lay& L = V.lay;
    const Off o(V.nu, V.nz);
    const int lane = threadIdx.x & 31;
    const int64_t bs = V.sl.base;
    if (i >= 1) {
        double* pv = y + (L.off_v(i) - bs);
        double* pm = y + (L.off_mu(i) - bs);
        for (int e = lane; e < V.nu; e += 32) { pv[e] = s[o.v + e]; pm[e] = s[o.m + e]; }
    }
    if (i < L.N) {
        double* pu = y + (L.off_u(i) - bs);
        double* pz = y + (L.off_z(i) - bs);
        double* pl = y + (L.off_l(i) - bs);
        for (int e = lane; e < V.nu; e += 32) { pu[e] = s[o.u + e]; pl[e] = s[o.l + e]; }
        for (int e = lane; e < V.nz; e += 32) pz[e] = s[o.z + e];
    }
}

// y = (A x)_i (kkt.py:228-247) with the continuity couplings uprev / munext
__device__ void apply_row(const GView& V, int i, const double* x, const double* uprev,
                          const double* munext, double* y) {
    const Lay& L = V.lay;
    const int nu = V.nu, nz = V.nz;
    const Off o(nu, nz);
    const int lane = threadIdx.x & 31;
    const bool has_vm = i >= 1, has_uzl = i < L.N;
    for (int e = lane; e < o.len; e += 32) y[e] = 0.0;
    __syncwarp();
    if (has_vm) {
        const double* Qv = (i == L.N) ? V.Ql : V.Qm;
        const double* C = has_uzl ? V.Ci(i) : nullptr;
        for (int e = lane; e < nu; e += 32) {
            double a = 0.0;
            for (int c = 0; c < nu; ++c) a += Qv[e * nu + c] * x[o.v + c];
            a -= x[o.m + e];
            if (C)
                for (int r = 0; r < nu; ++r) a += C[r * nu + e] * x[o.l + r];   // C^T lam
            y[o.v + e] = a;
            y[o.m + e] = -x[o.v + e] + (uprev ? uprev[e] : 0.0);
        }
    }
    if (has_uzl) {
        const double* Qu = (i == L.N - 1) ? V.Ql : V.Qm;
        const double* K = V.Ki(i);
        const double* B = V.Bi(i);
        const double* C = has_vm ? V.Ci(i) : nullptr;
        for (int e = lane; e < nu; e += 32) {
            double a = 0.0, l = 0.0;
            for (int c = 0; c < nu; ++c) {
                a += Qu[e * nu + c] * x[o.u + c] + K[c * nu + e] * x[o.l + c];   // Qu u + K^T lam
                l += K[e * nu + c] * x[o.u + c];                                   // K u
                if (C) l += C[e * nu + c] * x[o.v + c];                            // C v
            }
            for (int c = 0; c < nz; ++c) l += B[e * nz + c] * x[o.z + c];          // B z
            if (munext) a += munext[e];
            y[o.u + e] = a;
            y[o.l + e] = l;
        }
        for (int e = lane; e < nz; e += 32) {
            double a = 0.0;
            for (int c = 0; c < nz; ++c) a += V.Qz[e * nz + c] * x[o.z + c];
            for (int r = 0; r < nu; ++r) a += B[r * nz + e] * x[o.l + r];          // B^T lam
            y[o.z + e] = a;
        }
    }
    __syncwarp();
}

__device__ __forceinline__ double warp_sum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// d = D_i^{-1} r; A: m x (m+1) scratch, m = 2nu + nz
__device__ void solve_row(const GView& V, int i, const double* r, double* d, double* A) {
    const Lay& L = V.lay;
    const int nu = V.nu, nz = V.nz;
    const Off o(nu, nz);
    const int lane = threadIdx.x & 31;
    const bool has_vm = i >= 1, has_uzl = i < L.N;
    for (int e = lane; e < o.len; e += 32) d[e] = 0.0;
    __syncwarp();
    if (has_vm)
        for (int e = lane; e < nu; e += 32) d[o.v + e] = -r[o.m + e];
    __syncwarp();
    if (has_uzl) {
        const int m = 2 * nu + nz, ld = m + 1;
        const double* Qu = (i == L.N - 1) ? V.Ql : V.Qm;
        const double* K = V.Ki(i);
        const double* B = V.Bi(i);
        for (int e = lane; e < m * ld; e += 32) A[e] = 0.0;
        __syncwarp();
        for (int e = lane; e < nu * nu; e += 32) {
            const int rr = e / nu, c = e - rr * nu;
            A[rr * ld + c] = Qu[e];                    // Qu
            A[(nu + nz + rr) * ld + c] = K[e];         // K
            A[c * ld + nu + nz + rr] = K[e];           // K^T
        }
        for (int e = lane; e < nz * nz; e += 32) {
            const int rr = e / nz, c = e - rr * nz;
            A[(nu + rr) * ld + nu + c] = V.Qz[e];
        }
        for (int e = lane; e < nu * nz; e += 32) {
            const int rr = e / nz, c = e - rr * nz;    // B[rr][c]
            A[(nu + nz + rr) * ld + nu + c] = B[e];    // B
            A[(nu + c) * ld + nu + nz + rr] = B[e];    // B^T
        }
        __syncwarp();
        const double* C = has_vm ? V.Ci(i) : nullptr;
        for (int e = lane; e < nu; e += 32) {
            A[e * ld + m] = r[o.u + e];
            double g = r[o.l + e];
            if (C)
                for (int c = 0; c < nu; ++c) g -= C[e * nu + c] * d[o.v + c];
            A[(nu + nz + e) * ld + m] = g;
        }
        for (int e = lane; e < nz; e += 32) A[(nu + e) * ld + m] = r[o.z + e];
        __syncwarp();
        // Gaussian elimination with partial pivoting
        for (int k = 0; k < m; ++k) {
            double best = -1.0;
            int p = k;
            for (int rr = k + lane; rr < m; rr += 32) {
                const double v = fabs(A[rr * ld + k]);
                if (v > best) { best = v; p = rr; }
            }
            for (int off = 16; off > 0; off >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, off);
                const int op = __shfl_xor_sync(0xffffffffu, p, off);
                if (ob > best || (ob == best && op < p)) { best = ob; p = op; }
            }
            if (p != k)
                for (int c = k + lane; c <= m; c += 32) {
                    const double t = A[k * ld + c];
                    A[k * ld + c] = A[p * ld + c];
                    A[p * ld + c] = t;
                }
            __syncwarp();
            const double inv = 1.0 / A[k * ld + k];
            for (int rr = k + 1 + lane; rr < m; rr += 32) {
                const double f = A[rr * ld + k] * inv;
                for (int c = k + 1; c <= m; ++c) A[rr * ld + c] -= f * A[k * ld + c];
            }
            __syncwarp();
        }
        // back substitution; the solution overwrites the rhs column
        for (int k = m - 1; k >= 0; --k) {
            double s = 0.0;
            for (int c = k + 1 + lane; c < m; c += 32) s += A[k * ld + c] * A[c * ld + m];
            s = warp_sum(s);
            if (lane == 0) A[k * ld + m] = (A[k * ld + m] - s) / A[k * ld + k];
            __syncwarp();
        }
        for (int e = lane; e < nu; e += 32) {
            d[o.u + e] = A[e * ld + m];
            d[o.l + e] = A[(nu + nz + e) * ld + m];
        }
        for (int e = lane; e < nz; e += 32) d[o.z + e] = A[(nu + e) * ld + m];
        __syncwarp();
    }
    if (has_vm) {
        const double* Qv = (i == L.N) ? V.Ql : V.Qm;
        const double* C = has_uzl ? V.Ci(i) : nullptr;
        for (int e = lane; e < nu; e += 32) {
            double a = -r[o.v + e];
            for (int c = 0; c < nu; ++c) a += Qv[e * nu + c] * d[o.v + c];
            if (C)
                for (int rr = 0; rr < nu; ++rr) a += C[rr * nu + e] * d[o.l + rr];   // C^T lam
            d[o.m + e] = a;
        }
    }
    __syncwarp();
}

}  // namespace

// one warp (CTA of 32 threads) per block row; shared: x, y, b rows + A
template <int MODE>
__global__ void __launch_bounds__(32) denseg_rows(GView V, const double* __restrict__ b,
                                                  const double* __restrict__ x,
                                                  double* __restrict__ y, double omega) {
    extern __shared__ double gsm[];
    const Lay& L = V.lay;
    const Off o(V.nu, V.nz);
    double* xs = gsm;
    double* ys = xs + o.len;
    double* bs = ys + o.len;
    double* A = bs + o.len;
    const int lane = threadIdx.x;
    for (int i = V.sl.r0 + blockIdx.x; i < V.sl.r1; i += gridDim.x) {
        if (MODE == G_SOLVE) {
            load_row(V, i, b, bs);
            solve_row(V, i, bs, ys, A);
            store_row(V, i, y, ys);
            __syncwarp();
            continue;
        }
        const double* uprev = (MODE != G_APPLY_DIAG && x) ? V.sl.uprev(L, x, i) : nullptr;
        const double* munext = (MODE != G_APPLY_DIAG && x) ? V.sl.munext(L, x, i) : nullptr;
        load_row(V, i, x, xs);
        apply_row(V, i, xs, uprev, munext, ys);
        if (MODE == G_APPLY || MODE == G_APPLY_DIAG) {
            store_row(V, i, y, ys);
            __syncwarp();
            continue;
        }
        load_row(V, i, b, bs);
        for (int e = lane; e < o.len; e += 32) bs[e] -= ys[e];
        __syncwarp();
        if (MODE == G_RESIDUAL) {
            store_row(V, i, y, bs);
            __syncwarp();
            continue;
        }
        solve_row(V, i, bs, ys, A);   // x + omega D^{-1}(b - A x)
        for (int e = lane; e < o.len; e += 32) xs[e] += omega * ys[e];
        __syncwarp();
        store_row(V, i, y, xs);
        __syncwarp();
    }
}

// Serial block substitution (smoothers.py:79-109): (D - L) d = r walks the rows
// upwards with u_{i-1} of the previous row, (D - U) d = r downwards with mu_{i+1}.
template <bool FWD>
__global__ void __launch_bounds__(32) denseg_subst(GView V, const double* __restrict__ r,
                                                   double* __restrict__ d) {
    extern __shared__ double gsm[];
    const Lay& L = V.lay;
    const Off o(V.nu, V.nz);
    double* rs = gsm;
    double* ds = rs + o.len;
    double* cp = ds + o.len;           // coupling segment of the previous row (nu)
    double* A = cp + V.nu;
    const int lane = threadIdx.x;
    for (int s = 0; s <= L.N; ++s) {
        const int i = FWD ? s : L.N - s;
        load_row(V, i, r, rs);
        if (s > 0) {
            if (FWD) { for (int e = lane; e < V.nu; e += 32) rs[o.m + e] -= cp[e]; }
            else     { for (int e = lane; e < V.nu; e += 32) rs[o.u + e] -= cp[e]; }
        }
        __syncwarp();
        solve_row(V, i, rs, ds, A);
        store_row(V, i, d, ds);
        for (int e = lane; e < V.nu; e += 32) cp[e] = FWD ? ds[o.u + e] : ds[o.m + e];
        __syncwarp();
    }
}

bool denseg_supported(const tk_level* Lv) {
    return Lv->n_u >= 1 && Lv->n_u <= TK_MAX_DENSE_GENERAL && Lv->n_z >= 1 && Lv->n_z <= 8;
}

int denseg_launch(const tk_level* Lv, int op, const double* b, const double* x, double* y,
                  double omega, cudaStream_t s) {
    if (!denseg_supported(Lv)) {
        set_error("dense family supports n_u <= %d, n_z <= 8 (got n_u=%d n_z=%d)",
                  TK_MAX_DENSE_GENERAL, Lv->n_u, Lv->n_z);
        return TK_ERR_UNSUPPORTED;
    }
    GView V(Lv);
    const int rows = V.sl.r1 - V.sl.r0;
    const int nu = Lv->n_u, nz = Lv->n_z, m = 2 * nu + nz, len = 4 * nu + nz;
    const size_t smem = (size_t)(3 * len + nu + m * (m + 1)) * sizeof(double);
    static bool attr = false;
    if (!attr) {
        const int mx = 200 * 1024;
        cudaFuncSetAttribute(denseg_rows<G_APPLY>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(denseg_rows<G_APPLY_DIAG>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(denseg_rows<G_RESIDUAL>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(denseg_rows<G_SOLVE>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(denseg_rows<G_JACOBI>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(denseg_subst<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(denseg_subst<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_status(e, "denseg: cudaFuncSetAttribute");
        attr = true;
    }
    const int grid = rows < 148 * 16 ? rows : 148 * 16;
    if (op >= 10 && !V.sl.whole(Lv->n_steps)) {
        set_error("block Gauss-Seidel substitution needs the whole level (no time slab)");
        return TK_ERR_ARG;
    }
    switch (op) {
        case G_APPLY: denseg_rows<G_APPLY><<<grid, 32, smem, s>>>(V, b, x, y, omega); break;
        case G_APPLY_DIAG: denseg_rows<G_APPLY_DIAG><<<grid, 32, smem, s>>>(V, b, x, y, omega); break;
        case G_RESIDUAL: denseg_rows<G_RESIDUAL><<<grid, 32, smem, s>>>(V, b, x, y, omega); break;
        case G_SOLVE: denseg_rows<G_SOLVE><<<grid, 32, smem, s>>>(V, b, x, y, omega); break;
        case G_JACOBI: denseg_rows<G_JACOBI><<<grid, 32, smem, s>>>(V, b, x, y, omega); break;
        case 10: denseg_subst<true><<<1, 32, smem, s>>>(V, b, y); break;
        case 11: denseg_subst<false><<<1, 32, smem, s>>>(V, b, y); break;
        default:
            set_error("dense family (general sizes): op %d is not available", op);
            return TK_ERR_UNSUPPORTED;
    }
    return check_launch("denseg_rows");
}

}  // namespace tk
