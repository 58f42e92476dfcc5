// Krylov vector kernels for the device-resident (F)GMRES (krylov.py:77-191).
// Reductions are deterministic: a fixed grid of kReduceBlocks CTAs, each
// summing a fixed grid-stride slice, then one CTA summing the partials in a
// fixed tree order, so repeated solves are bitwise reproducible.
#include <cooperative_groups.h>
#include <stdlib.h>

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

// Krylov updates whose scalar lives in device memory (the sharded (F)GMRES:
// the scalar is an NCCL-allreduced dot that never visits the host).
__global__ void axpy_dev_kernel(int64_t n, const double* __restrict__ a, double sign,
                                const double* __restrict__ x, double* __restrict__ y) {
    const double c = sign * a[0];
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += stride)
        y[k] = fma(c, x[k], y[k]);
}

__global__ void sqrt_div_kernel(int64_t n, const double* __restrict__ sq, double* __restrict__ nrm,
                                const double* __restrict__ x, double* __restrict__ y) {
    const double s = sqrt(sq[0]);
    if (blockIdx.x == 0 && threadIdx.x == 0 && nrm) nrm[0] = s;
    if (s == 0.0 || !y) return;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += stride)
        y[k] = x[k] / s;
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

// ---------------------------------------------------------------------------
// One modified Gram-Schmidt Arnoldi step in a single cooperative launch
// (krylov.py:77-191, the inner `for i in range(j+1)` loop, the norm and the
// normalisation of the next basis vector):
//   for i = 0..j:  h_i = <V_i, w>;  w -= h_i V_i
//   h_{j+1} = ||w||;  V_{j+1} = (1 / h_{j+1}) w
// Pass i fuses the update with h_{i-1} into the reduction for h_i, so the
// sequential MGS chain costs one grid barrier per basis vector instead of a
// dot launch, a host round trip and an axpy launch.  The grid (kReduceBlocks
// CTAs of kReduceThreads), the per-thread element order, the two accumulators
// and the reduction trees are exactly those of dot_partial/sum_partials and
// axpy_kernel's fma, so h and w are bitwise identical to the unfused
// sequence tk_dot / tk_axpy / tk_nrm2 / tk_scale_into.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_xor_sum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// sum_partials' tree (1024 threads = 32 virtual warps) evaluated by one CTA
__device__ __forceinline__ double reduce_partials(const double* __restrict__ part, double* sh) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    constexpr int NW = kReduceThreads / 32;
    for (int vw = w; vw < 32; vw += NW) {
        const int k = 32 * vw + l;
        double v = k < kReduceBlocks ? __ldcg(part + k) : 0.0;
        v = warp_xor_sum(v);
        if (l == 0) sh[vw] = v;
    }
    __syncthreads();
    double r = 0.0;
    if (w == 0) {
        r = warp_xor_sum(sh[l]);
        if (l == 0) sh[32] = r;
    }
    __syncthreads();
    r = sh[32];
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(kReduceThreads, 4)
arnoldi_mgs_kernel(int64_t n, int j, double* __restrict__ V, int64_t ld, double* __restrict__ w,
                   double* __restrict__ h, double* __restrict__ part, const int* __restrict__ jdev,
                   int64_t hstride, double* __restrict__ vcopy) {
    namespace cg = cooperative_groups;
    if (jdev) {          // graphed GMRES: the step index lives on the device
        j = *jdev;
        h += (int64_t)j * hstride;
    }
    cg::grid_group grid = cg::this_grid();
    __shared__ double sh[kReduceThreads / 32 + 34];
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t k0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    double hp = 0.0;   // h_{i-1}
    for (int i = 0; i <= j + 1; ++i) {
        const double* Vp = i > 0 ? V + (int64_t)(i - 1) * ld : nullptr;   // update with h_{i-1}
        const double* Vi = i <= j ? V + (int64_t)i * ld : nullptr;         // dot against V_i (or w)
        const double a = -hp;
        double acc = 0.0, acc2 = 0.0;
        int64_t k = k0;
        // the basis vectors stream through L2 with evict-first loads so that w
        // (re-read and re-written every pass) stays L2-resident for large n
        for (; k + stride < n; k += 2 * stride) {
            double w0 = w[k], w1 = w[k + stride];
            if (Vp) {
                w0 = fma(a, __ldcs(Vp + k), w0);
                w1 = fma(a, __ldcs(Vp + k + stride), w1);
                w[k] = w0;
                w[k + stride] = w1;
            }
            acc = fma(Vi ? __ldcs(Vi + k) : w0, w0, acc);
            acc2 = fma(Vi ? __ldcs(Vi + k + stride) : w1, w1, acc2);
        }
        if (k < n) {
            double w0 = w[k];
            if (Vp) {
                w0 = fma(a, __ldcs(Vp + k), w0);
                w[k] = w0;
            }
            acc = fma(Vi ? __ldcs(Vi + k) : w0, w0, acc);
        }
        acc += acc2;
        // block_sum<kReduceThreads>
        acc = warp_xor_sum(acc);
        if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
        __syncthreads();
        double s = (threadIdx.x < kReduceThreads / 32) ? sh[threadIdx.x] : 0.0;
        if ((threadIdx.x >> 5) == 0) s = warp_xor_sum(s);
        double* pslot = part + (i & 1) * kReduceBlocks;
        if (threadIdx.x == 0) __stcg(pslot + blockIdx.x, s);
        __syncthreads();
        grid.sync();
        double hi = reduce_partials(pslot, sh);
        if (i == j + 1) hi = sqrt(hi);
        if (blockIdx.x == 0 && threadIdx.x == 0) h[i] = hi;
        hp = hi;
    }
    // V_{j+1} = (1 / h_{j+1}) w  (scale_into_kernel's a * x[k])
    if (hp != 0.0) {
        const double inv = 1.0 / hp;
        double* Vn = V + (int64_t)(j + 1) * ld;
        if (vcopy) {
            for (int64_t k = k0; k < n; k += stride) {
                const double v = inv * w[k];
                Vn[k] = v;
                vcopy[k] = v;
            }
        } else {
            for (int64_t k = k0; k < n; k += stride) Vn[k] = inv * w[k];
        }
    }
}

// w is re-read and re-written by every MGS pass while each basis vector is
// streamed once or twice: when w is too large to stay in L2 by itself next to
// the streamed basis (tens of MB), the launch marks it L2-persisting
// (access-policy window; the persisting carve-out is set once to the device
// maximum).  TK_ARNOLDI_PERSIST=0 disables it.
static bool g_persist_used = false;

struct PersistCap;
static void persist_release();
// nested solves: only the outermost one may hold w L2-persisting (the coarse
// GMRES inside a V-cycle inside an outer FGMRES would otherwise claim the
// carve-out for the whole outer solve)
static bool g_persist_allowed = true;
int l2_persist_allow(int on) {
    g_persist_allowed = on != 0;
    return TK_OK;
}

// return the persisting lines to normal status AND give the persisting
// carve-out back (host-synchronous: call after the stream that used the
// window has been synchronised, e.g. at the end of a Krylov solve).  The
// carve-out must not outlive the solve: while cudaLimitPersistingL2CacheSize
// is set, every later kernel runs in the remaining L2 only -- the n_u = 2048
// KKT apply of configs[4] took 5.96 ms instead of 3.32 ms after one coarse
// solve had left it set.
int l2_persist_reset() {
    if (!g_persist_used) return TK_OK;
    g_persist_used = false;
    const int e = cuda_status(cudaCtxResetPersistingL2Cache(), "cudaCtxResetPersistingL2Cache");
    persist_release();
    return e;
}

// Persisting-L2 budget of the current device: the window size and the
// persisting carve-out (set to the device maximum on first use), per device.
struct PersistCap {
    int64_t carve = -1;   // bytes of persisting L2 (0: unavailable / disabled)
    int64_t window = 0;   // max access-policy window
};
static PersistCap g_persist[64];

static PersistCap persist_cap() {
    int dev = 0;
    cudaGetDevice(&dev);
    PersistCap& c = g_persist[dev & 63];
    if (c.carve < 0) {
        c.carve = 0;
        const char* e = getenv("TK_ARNOLDI_PERSIST");
        if (e && e[0] == '0') return c;
        int mx = 0, win = 0;
        cudaDeviceGetAttribute(&mx, cudaDevAttrMaxPersistingL2CacheSize, dev);
        cudaDeviceGetAttribute(&win, cudaDevAttrMaxAccessPolicyWindowSize, dev);
        if (mx > 0 && win > 0 && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)mx) == cudaSuccess) {
            c.carve = mx;
            c.window = win;
        }
        cudaGetLastError();
    }
    return c;
}

static void persist_release() {
    int dev = 0;
    cudaGetDevice(&dev);
    PersistCap& c = g_persist[dev & 63];
    if (c.carve > 0) {
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0);
        cudaGetLastError();
        c.carve = -1;   // re-established by the next solve that wants it
    }
}

// Whether the fixed cooperative grid of the Arnoldi kernel is co-resident on
// the current device (not on a MIG slice / SM-limited MPS client / smaller
// part): checked once per device; the host falls back to the unfused kernels.
static int g_coop_ok[64];
int arnoldi_supported() {
    int dev = 0;
    cudaGetDevice(&dev);
    int& ok = g_coop_ok[dev & 63];
    if (ok == 0) {
        int sms = 0, per = 0, coop = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, arnoldi_mgs_kernel, kReduceThreads, 0);
        cudaGetLastError();
        ok = (coop && (int64_t)per * sms >= kReduceBlocks) ? 1 : -1;
    }
    return ok > 0;
}

int arnoldi_launch(int64_t n, int j, double* V, int64_t ld, double* w, double* h, double* work,
                   cudaStream_t s) {
    const int* jdev = nullptr;
    int64_t hstride = 0;
    double* vcopy = nullptr;
    if (!arnoldi_supported()) {
        set_error("tk_arnoldi_mgs: the cooperative grid of %d CTAs is not co-resident on this device",
                  kReduceBlocks);
        return TK_ERR_UNSUPPORTED;
    }
    const size_t wb = (size_t)n * 8;
    // w persisting only where most of it fits the carve-out (configs[3]: 75 MB);
    // far larger vectors (configs[2]: 335 MB) gain nothing and would only lose L2
    PersistCap pc = g_persist_allowed && wb >= ((size_t)16 << 20) && wb <= ((size_t)192 << 20) ? persist_cap()
                                                                           : PersistCap{0, 0};
    if (pc.carve > 0 && wb > 2 * (size_t)pc.carve) pc.carve = 0;
    if (pc.carve > 0) {
        // window over (the first window-size bytes of) w; the persisting
        // carve-out holds carve bytes of it
        const size_t nb = wb < (size_t)pc.window ? wb : (size_t)pc.window;
        const float hit = nb <= (size_t)pc.carve ? 1.0f : (float)pc.carve / (float)nb;
        g_persist_used = true;
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        at[1].id = cudaLaunchAttributeAccessPolicyWindow;
        at[1].val.accessPolicyWindow.base_ptr = (void*)w;
        at[1].val.accessPolicyWindow.num_bytes = nb;
        at[1].val.accessPolicyWindow.hitRatio = hit;
        at[1].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        at[1].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        cfg.gridDim = dim3(kReduceBlocks);
        cfg.blockDim = dim3(kReduceThreads);
        cfg.stream = s;
        cfg.attrs = at;
        cfg.numAttrs = 2;
        return cuda_status(cudaLaunchKernelEx(&cfg, arnoldi_mgs_kernel, n, j, V, ld, w, h, work, jdev,
                                              hstride, vcopy),
                           "arnoldi_mgs_kernel (persisting w)");
    }
    void* args[] = {(void*)&n, (void*)&j,    (void*)&V,       (void*)&ld,   (void*)&w,
                    (void*)&h, (void*)&work, (void*)&jdev, (void*)&hstride, (void*)&vcopy};
    const cudaError_t e = cudaLaunchCooperativeKernel((const void*)arnoldi_mgs_kernel,
                                                      dim3(kReduceBlocks), dim3(kReduceThreads),
                                                      args, 0, s);
    return cuda_status(e, "arnoldi_mgs_kernel");
}

// the step index j from device memory (*jdev), h = H + j*hstride, and the new
// basis vector also copied to vcopy (the next step's preconditioner input)
int arnoldi_dev_launch(int64_t n, const int* jdev, double* V, int64_t ld, double* w, double* H,
                       int64_t hstride, double* vcopy, double* work, cudaStream_t s) {
    if (!arnoldi_supported()) {
        set_error("tk_gm_arnoldi: the cooperative grid is not co-resident on this device");
        return TK_ERR_UNSUPPORTED;
    }
    int j = 0;
    void* args[] = {(void*)&n, (void*)&j,    (void*)&V,    (void*)&ld,      (void*)&w,
                    (void*)&H, (void*)&work, (void*)&jdev, (void*)&hstride, (void*)&vcopy};
    const cudaError_t e = cudaLaunchCooperativeKernel((const void*)arnoldi_mgs_kernel,
                                                      dim3(kReduceBlocks), dim3(kReduceThreads),
                                                      args, 0, s);
    return cuda_status(e, "arnoldi_mgs_kernel (device j)");
}

int64_t reduce_work_len() { return 2 * kReduceBlocks; }

// dst[k] = src[k] with SM loads/stores: used for the few Krylov scalars that
// cross between host and device through mapped pinned memory, so they never
// queue behind bulk copies on the copy engines (HostPipeline)
__global__ void copy_small_kernel(int64_t n, const double* __restrict__ src, double* __restrict__ dst) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        dst[k] = src[k];
}

int copy_small_launch(int64_t n, const double* src, double* dst, cudaStream_t s) {
    copy_small_kernel<<<grid_for(n, 256, 64), 256, 0, s>>>(n, src, dst);
    return check_launch("copy_small");
}

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

int axpy_dev_launch(int64_t n, const double* a, double sign, const double* x, double* y,
                    cudaStream_t s) {
    const int th = 256;
    axpy_dev_kernel<<<grid_for(n, th, 148 * 16), th, 0, s>>>(n, a, sign, x, y);
    return check_launch("axpy_dev");
}

int sqrt_div_launch(int64_t n, const double* sq, double* nrm, const double* x, double* y,
                    cudaStream_t s) {
    const int th = 256;
    sqrt_div_kernel<<<grid_for(n > 0 ? n : 1, th, 148 * 16), th, 0, s>>>(n, sq, nrm, x, y);
    return check_launch("sqrt_div");
}

int gemv_t_add_launch(int64_t n, int k, const double* V, int64_t ld, const double* c, double* x,
                      cudaStream_t s) {
    const int th = 256;
    gemv_t_add_kernel<<<grid_for(n, th, 148 * 16), th, 0, s>>>(n, k, V, ld, c, x);
    return check_launch("gemv_t_add");
}

}  // namespace tk
