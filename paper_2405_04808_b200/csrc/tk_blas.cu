// Krylov vector kernels for the device-resident (F)GMRES (krylov.py:77-191).
// Reductions are deterministic: a fixed grid of kReduceBlocks CTAs, each
// summing a fixed grid-stride slice, then one CTA summing the partials in a
// fixed tree order, so repeated solves are bitwise reproducible.
#include "tk_common.cuh"

namespace tk {

static constexpr int kReduceBlocks = 148 * 4;
static constexpr int kReduceThreads = 256;

template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) sh[w] = v;
    __syncthreads();
    v = (threadIdx.x < NT / 32) ? sh[threadIdx.x] : 0.0;
    if (w == 0) {
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    }
    return v;
}

__global__ void __launch_bounds__(kReduceThreads) dot_partial(int64_t n, const double* __restrict__ x,
                                                              const double* __restrict__ y,
                                                              double* __restrict__ part) {
    __shared__ double sh[kReduceThreads / 32];
    double acc = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    // 2-way unrolled, independent accumulators for ILP
    double acc2 = 0.0;
    for (; k + stride < n; k += 2 * stride) {
        acc = fma(x[k], y[k], acc);
        acc2 = fma(x[k + stride], y[k + stride], acc2);
    }
    if (k < n) acc = fma(x[k], y[k], acc);
    acc += acc2;
    double s = block_sum<kReduceThreads>(acc, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void __launch_bounds__(1024) sum_partials(int np, const double* __restrict__ part,
                                                     double* __restrict__ out, int take_sqrt) {
    __shared__ double sh[32];
    double v = 0.0;
    for (int k = threadIdx.x; k < np; k += blockDim.x) v += part[k];
    v = block_sum<1024>(v, sh);
    if (threadIdx.x == 0) *out = take_sqrt ? sqrt(v) : v;
}

__global__ void axpy_kernel(int64_t n, double a, const double* __restrict__ x,
                            double* __restrict__ y) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += stride)
        y[k] = fma(a, x[k], y[k]);
}

__global__ void scale_into_kernel(int64_t n, double a, const double* __restrict__ x,
                                  double* __restrict__ y) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += stride)
        y[k] = a * x[k];
}

__global__ void rsub_kernel(int64_t n, const double* __restrict__ b, double* __restrict__ y) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += stride)
        y[k] = b[k] - y[k];
}

__global__ void gemv_t_add_kernel(int64_t n, int kk, const double* __restrict__ V, int64_t ld,
                                  const double* __restrict__ c, double* __restrict__ x) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += stride) {
        double s = 0.0;
        for (int r = 0; r < kk; ++r) s = fma(c[r], V[(int64_t)r * ld + k], s);
        x[k] += s;
    }
}

int64_t reduce_work_len() { return kReduceBlocks; }

int dot_launch(int64_t n, const double* x, const double* y, double* out, double* work,
               int take_sqrt, cudaStream_t s) {
    dot_partial<<<kReduceBlocks, kReduceThreads, 0, s>>>(n, x, y, work);
    sum_partials<<<1, 1024, 0, s>>>(kReduceBlocks, work, out, take_sqrt);
    return check_launch("dot");
}

int vec_launch(int op, int64_t n, double a, const double* x, double* y, cudaStream_t s) {
    const int th = 256;
    const int g = grid_for(n, th, 148 * 16);
    switch (op) {
        case 0: axpy_kernel<<<g, th, 0, s>>>(n, a, x, y); break;
        case 1: scale_into_kernel<<<g, th, 0, s>>>(n, a, x, y); break;
        case 2: rsub_kernel<<<g, th, 0, s>>>(n, x, y); break;
        default: return TK_ERR_ARG;
    }
    return check_launch("vec");
}

int gemv_t_add_launch(int64_t n, int k, const double* V, int64_t ld, const double* c, double* x,
                      cudaStream_t s) {
    const int th = 256;
    gemv_t_add_kernel<<<grid_for(n, th, 148 * 16), th, 0, s>>>(n, k, V, ld, c, x);
    return check_launch("gemv_t_add");
}

}  // namespace tk
