// Definitions shared by the TRI-family translation units (tk_tri.cu,
// tk_tri_part.cu): padded node indexing, the level view and tridiagonal
// mat-vec helpers.
#pragma once

#include "tk_common.cuh"

namespace tk {

__host__ __device__ __forceinline__ constexpr int PI(int j) { return j + (j >> 4); }
__host__ __device__ __forceinline__ constexpr int padded(int n) { return n + (n >> 4) + 1; }
__host__ __device__ __forceinline__ constexpr int ilog2(int n) {
    return n <= 1 ? 0 : 1 + ilog2(n >> 1);
}

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
    Slab sl;
    const double* fac;   // factor records of the slab's stages (or null)
    const double* qzw;   // scalar reduced-system inverse at the cut (with fac)
    TView(const tk_level* L)
        : lay(L->n_steps, L->n_u, L->n_z), n(L->n_u), K(L->K), C(L->C), Qm(L->Qm), Ql(L->Ql),
          Qz(L->Qz), cr(L->qz_cr), kappa(L->kappa), sl(L, Lay(L->n_steps, L->n_u, L->n_z)),
          fac(L->fac), qzw(L->qz_w) {}
    // stage diagonals of global block row i (stage arrays start at the slab's first row)
    __device__ const double* Ki(int i, int n_) const { return K + (size_t)(i - sl.r0) * 3 * n_; }
    __device__ const double* Ci(int i, int n_) const { return C + (size_t)(i - sl.r0) * 3 * n_; }
};

template <int NT>
__device__ __forceinline__ int dimn(const TView& V) { return NT > 0 ? NT : V.n; }

// (A x)_j for a tridiagonal A stored [3][n] = (sub, diag, sup); x in global memory
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
// same with x in padded shared memory
__device__ __forceinline__ double tmv_s(const double* A, int n, const double* xs, int j) {
    double s = A[n + j] * xs[PI(j)];
    if (j > 0) s += A[j] * xs[PI(j - 1)];
    if (j < n - 1) s += A[2 * n + j] * xs[PI(j + 1)];
    return s;
}
__device__ __forceinline__ double tmtv_s(const double* A, int n, const double* xs, int j) {
    double s = A[n + j] * xs[PI(j)];
    if (j > 0) s += A[2 * n + j - 1] * xs[PI(j - 1)];
    if (j < n - 1) s += A[j + 1] * xs[PI(j + 1)];
    return s;
}

}  // namespace tk
