// CUDA-graph replay of a V-cycle whose coarse-grid GMRES runs as a
// device-side loop (reference multigrid.py:245-260 coarse_solve and
// krylov.py:77-191 gmres, from a zero initial guess).
//
// The host-driven coarse GMRES needs one host round trip per Arnoldi step
// (the Givens update and the stopping test) plus the initial norm, the
// coefficient upload and the true-residual check: the GPU drains and idles
// at every one of them.  Here the whole coarse solve is recorded once into a
// CUDA graph:
//
//   nrm2(b) -> gm_init (target, g_0, stop flag -> while condition)
//           -> V_0 = b / beta                          (scale_into's a * x)
//   WHILE (cond):  prec(v_j) -> A z_j -> MGS Arnoldi step (device j)
//                  -> gm_givens (rotations, |g_{j+1}|, breakdown / stop
//                     tests of krylov.py, cudaGraphSetConditional)
//   gm_combine: y = H^{-1} g (back substitution), vy = V^T y
//   prec(vy) -> x;  r = b - A x;  ||r||, ||x||  -> gm_finish
//
// gm_finish repeats the host's post-cycle tests (finite solution, breakdown
// with a non-zero residual, restart needed) and writes (flags, iterations)
// into mapped host memory.  Any flag means "take the eager path": the host
// re-runs the cycle with the host-driven solver, which reproduces the
// reference's behaviour for those rare cases exactly (restarts, basis
// growth, exceptions).  The arithmetic of every scalar step is the host's:
// products and sums are rounded separately (__dmul_rn/__dadd_rn, no FMA
// contraction) so the rotations match the Python-float Givens update.
#include <cuda_runtime.h>

#include "tk_common.cuh"

namespace tk {

int dot_launch(int64_t, const double*, const double*, double*, double*, int, cudaStream_t);
int vec_launch(int, int64_t, double, const double*, double*, cudaStream_t);
int arnoldi_dev_launch(int64_t n, const int* jdev, double* V, int64_t ld, double* w, double* H,
                       int64_t hstride, double* vcopy, double* work, cudaStream_t s);

namespace {

constexpr int kHead = 8;             // doubles of the state header
constexpr double kBreakdownTol = 1e-14;   // krylov.py BREAKDOWN_TOL
enum : int { GM_FALLBACK = 1, GM_BROKE = 2 };

struct GmHead {
    int j;          // Arnoldi steps taken in this cycle (next column index)
    int total;      // iterations of the solve
    int flags;
    int max_iters;
    double beta0, target, inv_beta, true_norm, x_norm, rel_tol;
};
static_assert(sizeof(GmHead) <= kHead * sizeof(double), "state header");

struct GmView {
    GmHead* hd;
    double* H;      // column j at H + j*(cap+1)
    double* g;      // cap+1
    double* cs;     // cap
    double* sn;     // cap
    double* y;      // cap
    int cap;
    __host__ __device__ GmView(double* st, int c) : cap(c) {
        hd = reinterpret_cast<GmHead*>(st);
        H = st + kHead;
        g = H + (int64_t)c * (c + 1);
        cs = g + c + 1;
        sn = cs + c;
        y = sn + c;
    }
};

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

__global__ void gm_init_kernel(double* st, int cap, double rel_tol, int max_iters,
                               cudaGraphConditionalHandle cond) {
    if (threadIdx.x != 0) return;
    GmView s(st, cap);
    const double beta = s.hd->beta0;
    int flags = 0;
    // beta == 0 (x = 0, no iteration), a non-finite norm (NonFiniteValue) and
    // max_iters <= 0 are left to the host path
    if (!(beta > 0.0) || !isfinite(beta) || max_iters <= 0) flags |= GM_FALLBACK;
    s.hd->j = 0;
    s.hd->total = 0;
    s.hd->flags = flags;
    s.hd->max_iters = max_iters;
    s.hd->rel_tol = rel_tol;
    s.hd->target = mul(rel_tol, beta);
    s.hd->inv_beta = 1.0 / beta;
    s.g[0] = beta;
    cudaGraphSetConditional(cond, flags ? 0u : 1u);
}

// V_0 = (1/beta) b and the first preconditioner input (scale_into_kernel's a * x)
__global__ void gm_scale_kernel(int64_t n, const double* __restrict__ b, const double* __restrict__ st,
                                double* __restrict__ V0, double* __restrict__ vj) {
    const double a = reinterpret_cast<const GmHead*>(st)->inv_beta;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += stride) {
        const double v = a * b[k];
        V0[k] = v;
        vj[k] = v;
    }
}

// Givens update of column j and the stopping tests (krylov.py:77-191; the
// host loop of paper_2405_04808_b200/krylov.py, operation for operation)
__global__ void gm_givens_kernel(double* st, int cap, cudaGraphConditionalHandle cond) {
    if (threadIdx.x != 0) return;
    GmView s(st, cap);
    GmHead& h = *s.hd;
    const int j = h.j;
    double* col = s.H + (int64_t)j * (cap + 1);
    bool stop = false;
    bool finite = true;
    for (int i = 0; i <= j + 1; ++i) finite = finite && isfinite(col[i]);
    if (!finite) {                       // NonFiniteValue on the host path
        h.flags |= GM_FALLBACK;
        cudaGraphSetConditional(cond, 0u);
        return;
    }
    const double hj1 = col[j + 1];
    for (int i = 0; i < j; ++i) {
        const double a = col[i], b = col[i + 1];
        col[i] = add(mul(s.cs[i], a), mul(s.sn[i], b));
        col[i + 1] = add(mul(-s.sn[i], a), mul(s.cs[i], b));
    }
    const double den = hypot(col[j], col[j + 1]);
    if (den == 0.0) {                    // Breakdown("zero diagonal in Givens elimination")
        h.flags |= GM_FALLBACK;
        cudaGraphSetConditional(cond, 0u);
        return;
    }
    s.cs[j] = col[j] / den;
    s.sn[j] = col[j + 1] / den;
    col[j] = den;
    col[j + 1] = 0.0;
    const double gj = s.g[j];
    s.g[j + 1] = mul(-s.sn[j], gj);
    s.g[j] = mul(s.cs[j], gj);
    h.total += 1;
    h.j = j + 1;
    const double est = fabs(s.g[j + 1]);
    if (hj1 <= mul(kBreakdownTol, h.beta0)) {
        h.flags |= GM_BROKE;
        stop = true;
    }
    if (est <= h.target || h.total >= h.max_iters) stop = true;
    if (!stop && j + 1 >= cap) {         // the host path grows the basis
        h.flags |= GM_FALLBACK;
        stop = true;
    }
    cudaGraphSetConditional(cond, stop ? 0u : 1u);
}

// y = H^{-1} g over the jd computed columns (krylov.py back substitution)
__global__ void gm_backsolve_kernel(double* st, int cap) {
    if (threadIdx.x != 0) return;
    GmView s(st, cap);
    const int jd = s.hd->j;
    const int64_t ld = cap + 1;
    for (int i = jd - 1; i >= 0; --i) {
        double acc = 0.0;
        for (int k = i + 1; k < jd; ++k) acc = add(acc, mul(s.H[k * ld + i], s.y[k]));
        s.y[i] = sub(s.g[i], acc) / s.H[i * ld + i];
    }
}

// vy = 0 * V_0 + V[:jd]^T y  (scale_into(0) then gemv_t_add_kernel's fma chain)
__global__ void gm_gemv_kernel(int64_t n, const double* __restrict__ V, int64_t ldv,
                               const double* __restrict__ st, int cap, double* __restrict__ vy) {
    GmView s(const_cast<double*>(st), cap);
    const int kk = s.hd->j;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += stride) {
        double acc = 0.0;
        for (int r = 0; r < kk; ++r) acc = fma(s.y[r], V[(int64_t)r * ldv + k], acc);
        vy[k] = add(mul(0.0, V[k]), acc);
    }
}

// Z[j] = z (j = the Arnoldi step about to run, read from the state)
__global__ void gm_storez_kernel(int64_t n, const double* __restrict__ z, double* __restrict__ Z,
                                 int64_t ldz, const double* __restrict__ st, int cap) {
    GmView s(const_cast<double*>(st), cap);
    const int j = s.hd->j;
    if (j < 0 || j >= cap) return;
    double* dst = Z + (int64_t)j * ldz;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += stride) dst[k] = z[k];
}

__global__ void gm_finish_kernel(double* st, int cap, int* res) {
    if (threadIdx.x != 0) return;
    GmView s(st, cap);
    GmHead& h = *s.hd;
    int flags = h.flags;
    const bool broke = (flags & GM_BROKE) != 0;
    if (!isfinite(h.x_norm)) flags |= GM_FALLBACK;
    const double tn = h.true_norm;
    const double bt = mul(mul(10.0, kBreakdownTol), h.beta0);
    if (broke && tn > fmax(h.target, bt)) flags |= GM_FALLBACK;
    if (!(tn <= h.target || h.total >= h.max_iters || broke)) flags |= GM_FALLBACK;   // restart
    h.flags = flags;
    res[0] = flags & GM_FALLBACK;
    res[1] = h.total;
    __threadfence_system();
}

}  // namespace

}  // namespace tk

using namespace tk;

extern "C" {

int tk_graph_capture_begin(void* stream) {
    TK_CHECK_ARG(stream, "tk_graph_capture_begin: capture needs a non-default stream");
    return cuda_status(cudaStreamBeginCapture(as_stream(stream), cudaStreamCaptureModeRelaxed),
                       "cudaStreamBeginCapture");
}

int tk_graph_cond_create(void* stream, uint64_t* handle) {
    TK_CHECK_ARG(stream && handle, "tk_graph_cond_create: bad arguments");
    cudaStreamCaptureStatus st;
    cudaGraph_t g = nullptr;
    int rc = cuda_status(cudaStreamGetCaptureInfo(as_stream(stream), &st, nullptr, &g, nullptr, nullptr),
                         "cudaStreamGetCaptureInfo");
    if (rc) return rc;
    if (st != cudaStreamCaptureStatusActive || !g) {
        set_error("tk_graph_cond_create: stream is not capturing");
        return TK_ERR_ARG;
    }
    cudaGraphConditionalHandle h;
    rc = cuda_status(cudaGraphConditionalHandleCreate(&h, g, 1u, cudaGraphCondAssignDefault),
                     "cudaGraphConditionalHandleCreate");
    if (rc) return rc;
    *handle = (uint64_t)h;
    return TK_OK;
}

// Append a WHILE node on `handle` to the graph captured on `stream` and start
// capturing its body on `body_stream`.
int tk_graph_while_begin(void* stream, void* body_stream, uint64_t handle) {
    TK_CHECK_ARG(stream && body_stream, "tk_graph_while_begin: bad arguments");
    cudaStreamCaptureStatus st;
    cudaGraph_t g = nullptr;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    int rc = cuda_status(cudaStreamGetCaptureInfo(as_stream(stream), &st, nullptr, &g, &deps, &nd),
                         "cudaStreamGetCaptureInfo");
    if (rc) return rc;
    if (st != cudaStreamCaptureStatusActive) {
        set_error("tk_graph_while_begin: stream is not capturing");
        return TK_ERR_ARG;
    }
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = (cudaGraphConditionalHandle)handle;
    p.conditional.type = cudaGraphCondTypeWhile;
    p.conditional.size = 1;
    cudaGraphNode_t node;
    rc = cuda_status(cudaGraphAddNode(&node, g, deps, nd, &p), "cudaGraphAddNode(while)");
    if (rc) return rc;
    rc = cuda_status(cudaStreamUpdateCaptureDependencies(as_stream(stream), &node, 1,
                                                         cudaStreamSetCaptureDependencies),
                     "cudaStreamUpdateCaptureDependencies");
    if (rc) return rc;
    cudaGraph_t body = p.conditional.phGraph_out[0];
    return cuda_status(cudaStreamBeginCaptureToGraph(as_stream(body_stream), body, nullptr, nullptr, 0,
                                                     cudaStreamCaptureModeRelaxed),
                       "cudaStreamBeginCaptureToGraph(body)");
}

int tk_graph_while_end(void* body_stream) {
    cudaGraph_t g = nullptr;
    return cuda_status(cudaStreamEndCapture(as_stream(body_stream), &g), "cudaStreamEndCapture(body)");
}

int tk_graph_capture_end(void* stream, void** exec) {
    TK_CHECK_ARG(stream && exec, "tk_graph_capture_end: bad arguments");
    cudaGraph_t g = nullptr;
    int rc = cuda_status(cudaStreamEndCapture(as_stream(stream), &g), "cudaStreamEndCapture");
    if (rc) return rc;
    cudaGraphExec_t e = nullptr;
    rc = cuda_status(cudaGraphInstantiate(&e, g, 0), "cudaGraphInstantiate");
    cudaGraphDestroy(g);
    if (rc) return rc;
    *exec = (void*)e;
    return TK_OK;
}

int tk_graph_launch(void* exec, void* stream) {
    TK_CHECK_ARG(exec, "tk_graph_launch: null graph");
    return cuda_status(cudaGraphLaunch((cudaGraphExec_t)exec, as_stream(stream)), "cudaGraphLaunch");
}

int tk_graph_destroy(void* exec) {
    if (!exec) return TK_OK;
    return cuda_status(cudaGraphExecDestroy((cudaGraphExec_t)exec), "cudaGraphExecDestroy");
}

int64_t tk_gm_state_len(int32_t cap) {
    if (cap < 1) return -1;
    return kHead + (int64_t)cap * (cap + 1) + (cap + 1) + 3 * (int64_t)cap;
}

int tk_gm_begin(int64_t n, const double* b, double* V, int64_t ld, double* vj, double* state,
                int32_t cap, double rel_tol, int32_t max_iters, uint64_t handle, double* work,
                void* stream) {
    TK_CHECK_ARG(b && V && vj && state && work && n > 0 && ld >= n && cap >= 1,
                 "tk_gm_begin: bad arguments");
    cudaStream_t s = as_stream(stream);
    GmView v(state, cap);
    int rc = dot_launch(n, b, b, &v.hd->beta0, work, 1, s);
    if (rc) return rc;
    gm_init_kernel<<<1, 32, 0, s>>>(state, cap, rel_tol, max_iters, (cudaGraphConditionalHandle)handle);
    rc = check_launch("gm_init_kernel");
    if (rc) return rc;
    gm_scale_kernel<<<grid_for(n, 256, 148 * 16), 256, 0, s>>>(n, b, state, V, vj);
    return check_launch("gm_scale_kernel");
}

int tk_gm_arnoldi(int64_t n, double* V, int64_t ld, double* w, double* state, int32_t cap,
                  double* vj, double* work, void* stream) {
    TK_CHECK_ARG(V && w && state && work && n > 0 && ld >= n && cap >= 1,
                 "tk_gm_arnoldi: bad arguments");
    GmView v(state, cap);
    return arnoldi_dev_launch(n, &v.hd->j, V, ld, w, v.H, cap + 1, vj, work, as_stream(stream));
}

int tk_gm_storez(int64_t n, const double* z, double* Z, int64_t ldz, const double* state,
                 int32_t cap, void* stream) {
    TK_CHECK_ARG(z && Z && state && n > 0 && ldz >= n && cap >= 1, "tk_gm_storez: bad arguments");
    gm_storez_kernel<<<grid_for(n, 256, 148 * 16), 256, 0, as_stream(stream)>>>(n, z, Z, ldz, state, cap);
    return check_launch("gm_storez_kernel");
}

int tk_gm_givens(double* state, int32_t cap, uint64_t handle, void* stream) {
    TK_CHECK_ARG(state && cap >= 1, "tk_gm_givens: bad arguments");
    gm_givens_kernel<<<1, 32, 0, as_stream(stream)>>>(state, cap, (cudaGraphConditionalHandle)handle);
    return check_launch("gm_givens_kernel");
}

int tk_gm_combine(int64_t n, const double* V, int64_t ld, double* state, int32_t cap, double* vy,
                  void* stream) {
    TK_CHECK_ARG(V && state && vy && n > 0 && ld >= n && cap >= 1, "tk_gm_combine: bad arguments");
    cudaStream_t s = as_stream(stream);
    gm_backsolve_kernel<<<1, 32, 0, s>>>(state, cap);
    int rc = check_launch("gm_backsolve_kernel");
    if (rc) return rc;
    gm_gemv_kernel<<<grid_for(n, 256, 148 * 16), 256, 0, s>>>(n, V, ld, state, cap, vy);
    return check_launch("gm_gemv_kernel");
}

// r holds A x on entry: r = b - A x, ||r||, ||x||, then the host's post-cycle tests
int tk_gm_finish(int64_t n, const double* b, double* r, const double* x, double* state,
                 int32_t cap, int32_t* res, double* work, void* stream) {
    TK_CHECK_ARG(b && r && x && state && res && work && n > 0 && cap >= 1,
                 "tk_gm_finish: bad arguments");
    cudaStream_t s = as_stream(stream);
    GmView v(state, cap);
    int rc = vec_launch(2, n, 0.0, b, r, s);
    if (rc) return rc;
    rc = dot_launch(n, x, x, &v.hd->x_norm, work, 1, s);
    if (rc) return rc;
    rc = dot_launch(n, r, r, &v.hd->true_norm, work, 1, s);
    if (rc) return rc;
    gm_finish_kernel<<<1, 32, 0, s>>>(state, cap, res);
    return check_launch("gm_finish_kernel");
}

}  // extern "C"
