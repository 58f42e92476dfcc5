// Shared device/host helpers for the tempokkt_b200 kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "tempokkt_b200.h"

namespace tk {

void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* where);
int check_launch(const char* where);

#define TK_CHECK_ARG(cond, msg)            \
    do {                                   \
        if (!(cond)) {                     \
            ::tk::set_error("%s", msg);    \
            return TK_ERR_ARG;             \
        }                                  \
    } while (0)

// Reference time-clustered layout (kkt.py:127-191).  Block 0 = (u,z,lam),
// blocks 1..N-1 = (v,u,z,mu,lam), block N = (v,mu).
struct Lay {
    int N, nu, nz;
    int64_t F, m;
    __host__ __device__ Lay(int N_, int nu_, int nz_)
        : N(N_), nu(nu_), nz(nz_), F(2 * nu_ + nz_), m(4 * nu_ + nz_) {}
    __host__ __device__ int64_t dim() const { return (int64_t)N * m; }
    __host__ __device__ int64_t start(int i) const {
        return i == 0 ? 0 : F + (int64_t)(i - 1) * m;
    }
    // segment offsets of block row i; -1 when the block has no such segment
    __host__ __device__ int64_t off_v(int i) const { return i >= 1 ? start(i) : -1; }
    __host__ __device__ int64_t off_u(int i) const {
        return i == 0 ? 0 : (i < N ? start(i) + nu : -1);
    }
    __host__ __device__ int64_t off_z(int i) const {
        return i == 0 ? nu : (i < N ? start(i) + 2 * nu : -1);
    }
    __host__ __device__ int64_t off_mu(int i) const {
        return i == N ? start(i) + nu : (i >= 1 ? start(i) + 2 * nu + nz : -1);
    }
    __host__ __device__ int64_t off_l(int i) const {
        return i == 0 ? nu + nz : (i < N ? start(i) + 3 * nu + nz : -1);
    }
    // time-index (1-based) offsets of each variable kind
    __host__ __device__ int64_t t_u(int t) const { return off_u(t - 1); }
    __host__ __device__ int64_t t_z(int t) const { return off_z(t - 1); }
    __host__ __device__ int64_t t_l(int t) const { return off_l(t - 1); }
    __host__ __device__ int64_t t_v(int t) const { return off_v(t); }
    __host__ __device__ int64_t t_mu(int t) const { return off_mu(t); }
};

// Time slab of a level: global block rows [r0, r1); local vectors start at the
// global offset `base` of row r0; stage arrays start at stage r0; hu / hm are
// the halo u-segment of row r0-1 and mu-segment of row r1.
struct Slab {
    int r0, r1;
    int64_t base;
    const double* hu;
    const double* hm;
    __host__ Slab(const tk_level* L, const Lay& lay)
        : r0(L->row0), r1(L->row1 > 0 ? L->row1 : L->n_steps + 1), base(lay.start(L->row0)),
          hu(L->halo_u), hm(L->halo_mu) {}
    __host__ __device__ bool whole(int N) const { return r0 == 0 && r1 == N + 1; }
    // coupling sources of row i for a local vector x (nullptr when absent)
    __host__ __device__ const double* uprev(const Lay& L, const double* x, int i) const {
        if (i < 1) return nullptr;
        return (i - 1 >= r0) ? x + (L.off_u(i - 1) - base) : hu;
    }
    __host__ __device__ const double* munext(const Lay& L, const double* x, int i) const {
        if (i >= L.N) return nullptr;
        return (i + 1 < r1) ? x + (L.off_mu(i + 1) - base) : hm;
    }
};

inline int grid_for(int64_t n, int threads, int cap = 148 * 16) {
    int64_t g = (n + threads - 1) / threads;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (int)g;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

}  // namespace tk
