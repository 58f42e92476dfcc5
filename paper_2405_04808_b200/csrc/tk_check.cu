// Setup-time singularity checks of the stage data (one pass per level, not
// on the hot path):
//
//  * tk_check_k      -- the K_i half of Theorem 1 (check_theorem1,
//    kkt.py:530-543): K_i is "singular" when partial-pivoting LU
//    (linalg.lu_factor, linalg.py:75-103, i.e. LAPACK getrf) meets a pivot
//    below pivot_floor * max|K_i| or K_i has a non-finite entry.  TRI stages
//    run the tridiagonal elimination with the same row interchanges as dense
//    GEPP (a row below i+1 never holds a nonzero in column i, so getrf on a
//    tridiagonal matrix only ever compares rows i and i+1 -- LAPACK gttrf).
//    DENSE stages run getrf on the n_u x n_u block.
//  * tk_check_blocks -- the diagonal-block factorisation of DiagonalSolver
//    (kkt.py:347-368, the reference raises SingularBlock(i) there): DENSE
//    levels assemble each (4n_u+n_z)-wide diagonal block exactly as
//    assemble_kkt (kkt.py:279-320) and run getrf on it with the same floor.
//    TRI blocks are symmetric quasi-definite once the weights are SPD (the
//    host checks those), so they are nonsingular by construction.
//
// Output: one int32 flag per stage (tk_check_k) or per block row 0..N
// (tk_check_blocks), 1 = singular, computed by one thread each.
#include <math.h>

#include "tk_common.cuh"

namespace tk {

// getrf pivot test on an m x m row-major matrix in local memory; true when a
// pivot falls below floor*max|a| or an entry is not finite.
template <int MAXM>
__device__ bool getrf_singular(double* a, int m, double pivot_floor) {
    double scale = 0.0;
    for (int e = 0; e < m * m; ++e) {
        const double v = a[e];
        if (!isfinite(v)) return true;
        scale = fmax(scale, fabs(v));
    }
    const double floor_ = pivot_floor * fmax(scale, 1e-300);
    for (int k = 0; k < m; ++k) {
        int p = k;                       // idamax: first index of the largest |a_rk|
        double best = fabs(a[k * m + k]);
        for (int r = k + 1; r < m; ++r) {
            const double v = fabs(a[r * m + k]);
            if (v > best) { best = v; p = r; }
        }
        if (best < floor_) return true;  // min |U_kk| below the floor
        if (p != k)
            for (int c = 0; c < m; ++c) {
                const double t = a[k * m + c];
                a[k * m + c] = a[p * m + c];
                a[p * m + c] = t;
            }
        const double inv = 1.0 / a[k * m + k];
        for (int r = k + 1; r < m; ++r) {
            const double l = a[r * m + k] * inv;
            for (int c = k + 1; c < m; ++c) a[r * m + c] -= l * a[k * m + c];
        }
    }
    return false;
}

// Tridiagonal GEPP (gttrf) of K_i given as [3][n] (sub, diag, sup).
__device__ bool tri_singular(const double* K, int n, double pivot_floor) {
    const double* sub = K;
    const double* dia = K + n;
    const double* sup = K + 2 * n;
    double scale = 0.0;
    for (int j = 0; j < n; ++j) {
        const double a = dia[j];
        const double b = j > 0 ? sub[j] : 0.0;
        const double c = j < n - 1 ? sup[j] : 0.0;
        if (!isfinite(a) || !isfinite(b) || !isfinite(c)) return true;
        scale = fmax(scale, fmax(fabs(a), fmax(fabs(b), fabs(c))));
    }
    const double floor_ = pivot_floor * fmax(scale, 1e-300);
    double d = dia[0], du = n > 1 ? sup[0] : 0.0;   // current pivot row (cols i, i+1)
    for (int i = 0; i < n - 1; ++i) {
        const double l = sub[i + 1];                 // row i+1, col i
        double nd = dia[i + 1];                      // row i+1, col i+1
        double ndu = i + 1 < n - 1 ? sup[i + 1] : 0.0;
        if (fabs(d) >= fabs(l)) {                    // no interchange
            if (fabs(d) < floor_) return true;
            nd -= (l / d) * du;
        } else {                                     // rows i and i+1 swap
            if (fabs(l) < floor_) return true;
            const double f = d / l;
            const double t = du - f * nd;
            ndu = -f * ndu;
            nd = t;
        }
        d = nd;
        du = ndu;
    }
    return fabs(d) < floor_;
}

__global__ void check_k_kernel(tk_level L, int ns, double pivot_floor, int32_t* bad) {
    const int nu = L.n_u;
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < ns; s += gridDim.x * blockDim.x) {
        bool sing;
        if (L.family == TK_FAMILY_TRI) {
            sing = tri_singular(L.K + (size_t)s * 3 * nu, nu, pivot_floor);
        } else {
            double a[TK_MAX_DENSE * TK_MAX_DENSE];
            for (int e = 0; e < nu * nu; ++e) a[e] = L.K[(size_t)s * nu * nu + e];
            sing = getrf_singular<TK_MAX_DENSE>(a, nu, pivot_floor);
        }
        bad[s] = sing ? 1 : 0;
    }
}

constexpr int kMaxBlock = 4 * TK_MAX_DENSE + TK_MAX_DENSE;

// Diagonal block of block row i (kkt.py:279-320), DENSE stage data of the
// whole level.  Weights: q_u[s] = q_v[s] = Qm (s < N-1), Ql (s = N-1).
__device__ int dense_block(const tk_level& L, int i, double* a) {
    const int N = L.n_steps, nu = L.n_u, nz = L.n_z;
    auto Q = [&](int s) { return s < N - 1 ? L.Qm : L.Ql; };
    if (i == 0 || i == N) {
        const int m = (i == 0) ? 2 * nu + nz : 2 * nu;
        for (int e = 0; e < m * m; ++e) a[e] = 0.0;
        if (i == 0) {
            const double* K = L.K;
            const double* B = L.B;
            const double* qu = Q(0);
            for (int r = 0; r < nu; ++r)
                for (int c = 0; c < nu; ++c) {
                    a[r * m + c] = qu[r * nu + c];
                    a[r * m + nu + nz + c] = K[c * nu + r];          // K^T
                    a[(nu + nz + r) * m + c] = K[r * nu + c];        // K
                }
            for (int r = 0; r < nz; ++r) {
                for (int c = 0; c < nz; ++c) a[(nu + r) * m + nu + c] = L.Qz[r * nz + c];
                for (int c = 0; c < nu; ++c) {
                    a[(nu + r) * m + nu + nz + c] = B[c * nz + r];   // B^T
                    a[(nu + nz + c) * m + nu + r] = B[c * nz + r];   // B
                }
            }
        } else {
            const double* qv = Q(N - 1);
            for (int r = 0; r < nu; ++r) {
                for (int c = 0; c < nu; ++c) a[r * m + c] = qv[r * nu + c];
                a[r * m + nu + r] = -1.0;
                a[(nu + r) * m + r] = -1.0;
            }
        }
        return m;
    }
    const int m = 4 * nu + nz;
    const int iv = 0, iu = nu, iz = 2 * nu, imu = 2 * nu + nz, il = 3 * nu + nz;
    for (int e = 0; e < m * m; ++e) a[e] = 0.0;
    const double* K = L.K + (size_t)i * nu * nu;
    const double* Cm = L.C + (size_t)i * nu * nu;
    const double* B = L.B + (size_t)i * nu * nz;
    const double* qv = Q(i - 1);
    const double* qu = Q(i);
    for (int r = 0; r < nu; ++r)
        for (int c = 0; c < nu; ++c) {
            a[(iv + r) * m + iv + c] = qv[r * nu + c];
            a[(iu + r) * m + iu + c] = qu[r * nu + c];
            a[(iv + r) * m + il + c] = Cm[c * nu + r];
            a[(iu + r) * m + il + c] = K[c * nu + r];
            a[(il + r) * m + iv + c] = Cm[r * nu + c];
            a[(il + r) * m + iu + c] = K[r * nu + c];
        }
    for (int r = 0; r < nu; ++r) {
        a[(iv + r) * m + imu + r] = -1.0;
        a[(imu + r) * m + iv + r] = -1.0;
    }
    for (int r = 0; r < nz; ++r) {
        for (int c = 0; c < nz; ++c) a[(iz + r) * m + iz + c] = L.Qz[r * nz + c];
        for (int c = 0; c < nu; ++c) {
            a[(iz + r) * m + il + c] = B[c * nz + r];
            a[(il + c) * m + iz + r] = B[c * nz + r];
        }
    }
    return m;
}

__global__ void check_blocks_kernel(tk_level L, double pivot_floor, int32_t* bad) {
    const int N = L.n_steps;
    double a[kMaxBlock * kMaxBlock];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= N; i += gridDim.x * blockDim.x) {
        const int m = dense_block(L, i, a);
        bad[i] = getrf_singular<kMaxBlock>(a, m, pivot_floor) ? 1 : 0;
    }
}

// General DENSE sizes (n_u, n_z beyond TK_MAX_DENSE): the same getrf tests with
// the work matrix in shared memory, one CTA per stage / block row (setup only).
__global__ void check_k_big_kernel(tk_level L, int ns, double pivot_floor, int32_t* bad) {
    extern __shared__ double csm[];
    const int nu = L.n_u;
    for (int s = blockIdx.x; s < ns; s += gridDim.x) {
        if (threadIdx.x == 0) {
            for (int e = 0; e < nu * nu; ++e) csm[e] = L.K[(size_t)s * nu * nu + e];
            bad[s] = getrf_singular<0>(csm, nu, pivot_floor) ? 1 : 0;
        }
    }
}
__global__ void check_blocks_big_kernel(tk_level L, double pivot_floor, int32_t* bad) {
    extern __shared__ double csm[];
    for (int i = blockIdx.x; i <= L.n_steps; i += gridDim.x) {
        if (threadIdx.x == 0) {
            const int m = dense_block(L, i, csm);
            bad[i] = getrf_singular<0>(csm, m, pivot_floor) ? 1 : 0;
        }
    }
}
static bool dense_big(const tk_level* L) {
    return L->family == TK_FAMILY_DENSE && (L->n_u > TK_MAX_DENSE || L->n_z > TK_MAX_DENSE);
}

int check_k_launch(const tk_level* L, double pivot_floor, int32_t* bad, cudaStream_t s) {
    const int r1 = L->row1 > 0 ? L->row1 : L->n_steps + 1;
    const int ns = (r1 < L->n_steps ? r1 : L->n_steps) - L->row0;
    if (ns <= 0) return TK_OK;
    if (dense_big(L)) {
        const size_t sm = (size_t)L->n_u * L->n_u * sizeof(double);
        check_k_big_kernel<<<ns < 2048 ? ns : 2048, 32, sm, s>>>(*L, ns, pivot_floor, bad);
        return check_launch("check_k (general dense)");
    }
    check_k_kernel<<<grid_for(ns, 64, 148 * 32), 64, 0, s>>>(*L, ns, pivot_floor, bad);
    return check_launch("check_k");
}

int check_blocks_launch(const tk_level* L, double pivot_floor, int32_t* bad, cudaStream_t s) {
    if (dense_big(L)) {
        const int m = 4 * L->n_u + L->n_z;
        const size_t sm = (size_t)m * m * sizeof(double);
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(check_blocks_big_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 220 * 1024);
            attr = true;
        }
        const int rows = L->n_steps + 1;
        check_blocks_big_kernel<<<rows < 2048 ? rows : 2048, 32, sm, s>>>(*L, pivot_floor, bad);
        return check_launch("check_blocks (general dense)");
    }
    check_blocks_kernel<<<grid_for(L->n_steps + 1, 32, 148 * 64), 32, 0, s>>>(*L, pivot_floor,
                                                                             bad);
    return check_launch("check_blocks");
}

}  // namespace tk
