// extern "C" entry points of libtempokkt_b200.so (include/tempokkt_b200.h).
#include <stdarg.h>
#include <stdio.h>

#include "tk_common.cuh"

namespace tk {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int cuda_status(cudaError_t e, const char* where) {
    if (e == cudaSuccess) return TK_OK;
    set_error("%s: %s", where, cudaGetErrorString(e));
    return TK_ERR_CUDA;
}

int check_launch(const char* where) { return cuda_status(cudaGetLastError(), where); }

int dense_launch(const tk_level*, int, const double*, const double*, double*, double, cudaStream_t);
int tri_launch(const tk_level*, int, const double*, const double*, double*, double, cudaStream_t);
int64_t tri_smem_bytes(int n);
int tri_resrestrict_launch(const tk_level*, const double*, const double*, double*, cudaStream_t);
bool tri_jacobi0_restrict_ok(const tk_level*, double);
int tri_jacobi0_restrict_launch(const tk_level*, const double*, double, double*, double*, cudaStream_t,
                                int partial = 0);
bool tri_jacobi_prolong_ok(const tk_level*, double);
int tri_jacobi_restrict_launch(const tk_level*, const double*, const double*, double*, double*,
                               cudaStream_t);
int tri_jacobi_prolong_launch(const tk_level*, const double*, const double*, const double*, double*,
                              cudaStream_t, const double* chalo = nullptr);
int tri_restrict_fix_slab_launch(const tk_level*, double*, cudaStream_t, int phase = 0);
int dense_jacobi0_restrict(const tk_level*, const double*, double*, double*, cudaStream_t);
int dense_split(const tk_level*, const double*, const double*, double*, const double*, double*, int,
                cudaStream_t, const double* chalo = nullptr);
int64_t tri_fac_len(const tk_level*);
int64_t tri_scratch_len(const tk_level*);
int64_t dense_fac_len(const tk_level*);
int32_t tri_cut_nodes(int n);
int32_t tri_cut_level(int n);
int32_t tri_chain_chunk_default(int n, int N);
int64_t tri_chain_prod_len(const tk_level*);
int64_t dense_scratch_len(const tk_level*);
int transfer_launch(int, int, int, int, int, int, const double*, const double*, const double*,
                    double*, cudaStream_t);
int64_t reduce_work_len();
int dot_launch(int64_t, const double*, const double*, double*, double*, int, cudaStream_t);
int vec_launch(int, int64_t, double, const double*, double*, cudaStream_t);
int gemv_t_add_launch(int64_t, int, const double*, int64_t, const double*, double*, cudaStream_t);
int axpy_dev_launch(int64_t, const double*, double, const double*, double*, cudaStream_t);
int sqrt_div_launch(int64_t, const double*, double*, const double*, double*, cudaStream_t);
int arnoldi_launch(int64_t, int, double*, int64_t, double*, double*, double*, cudaStream_t);
int l2_persist_reset();
int l2_persist_allow(int);
int arnoldi_supported();
int copy_small_launch(int64_t, const double*, double*, cudaStream_t);
int restrict_jacobi0_launch(int, int, int, int, int, const double*, const double*, const double*,
                            const double*, double, double*, cudaStream_t);
int stage_vdp_launch(int, double, double, double, int, const double*, const double*,
                     const double*, const double*, double*, double*, double*, cudaStream_t);
int stage_burgers_launch(int, int, double, double, double, const double*, const double*,
                         const double*, double*, double*, cudaStream_t);
int check_k_launch(const tk_level*, double, int32_t*, cudaStream_t);
int check_blocks_launch(const tk_level*, double, int32_t*, cudaStream_t);

static int check_level(const tk_level* L) {
    if (!L) { set_error("null level"); return TK_ERR_ARG; }
    if (L->n_steps < 1 || L->n_u < 1 || L->n_z < 1) {
        set_error("bad level sizes N=%d nu=%d nz=%d", L->n_steps, L->n_u, L->n_z);
        return TK_ERR_ARG;
    }
    if (!L->K || !L->C || !L->Qm || !L->Ql || !L->Qz) {
        set_error("level is missing stage/weight data");
        return TK_ERR_ARG;
    }
    {
        const int r1 = L->row1 > 0 ? L->row1 : L->n_steps + 1;
        if (L->row0 < 0 || L->row0 >= r1 || r1 > L->n_steps + 1) {
            set_error("bad time slab [%d, %d) for N=%d", L->row0, L->row1, L->n_steps);
            return TK_ERR_ARG;
        }
        if ((L->row0 > 0 && !L->halo_u) || (r1 <= L->n_steps && !L->halo_mu)) {
            set_error("time slab [%d, %d) needs its halo buffers", L->row0, r1);
            return TK_ERR_ARG;
        }
    }
    if (L->family == TK_FAMILY_DENSE) {
        if (!L->B || !L->Qm_inv || !L->Ql_inv || !L->Qz_inv) {
            set_error("dense level is missing B or weight inverses");
            return TK_ERR_ARG;
        }
    } else if (L->family == TK_FAMILY_TRI) {
        if (!L->qz_cr) { set_error("tri level is missing qz_cr"); return TK_ERR_ARG; }
    } else {
        set_error("unknown family %d", L->family);
        return TK_ERR_UNSUPPORTED;
    }
    return TK_OK;
}

static int level_op(const tk_level* L, int dense_op, int tri_op, const double* b,
                    const double* x, double* y, double omega, void* stream) {
    int rc = check_level(L);
    if (rc) return rc;
    cudaStream_t s = as_stream(stream);
    if (L->family == TK_FAMILY_DENSE) return dense_launch(L, dense_op, b, x, y, omega, s);
    return tri_launch(L, tri_op, b, x, y, omega, s);
}

}  // namespace tk

using namespace tk;

extern "C" {

const char* tk_version(void) { return "tempokkt_b200 0.1 (sm_100a)"; }
const char* tk_last_error(void) { return g_err; }

int64_t tk_kkt_dim(int32_t n_steps, int32_t n_u, int32_t n_z) {
    return (int64_t)n_steps * (4 * (int64_t)n_u + n_z);
}

int64_t tk_tri_smem_bytes(int32_t n_u) { return tri_smem_bytes(n_u); }

int tk_kkt_apply(const tk_level* L, const double* x, double* y, void* stream) {
    TK_CHECK_ARG(x && y, "tk_kkt_apply: null vector");
    return level_op(L, 0, 0, nullptr, x, y, 1.0, stream);
}

int tk_kkt_apply_diag(const tk_level* L, const double* x, double* y, void* stream) {
    TK_CHECK_ARG(x && y, "tk_kkt_apply_diag: null vector");
    return level_op(L, 1, 1, nullptr, x, y, 1.0, stream);
}

int tk_kkt_residual(const tk_level* L, const double* b, const double* x, double* r,
                    void* stream) {
    TK_CHECK_ARG(b && x && r, "tk_kkt_residual: null vector");
    return level_op(L, 2, 2, b, x, r, 1.0, stream);
}

int tk_diag_solve(const tk_level* L, const double* r, double* y, void* stream) {
    TK_CHECK_ARG(r && y, "tk_diag_solve: null vector");
    return level_op(L, 3, 3, r, nullptr, y, 1.0, stream);
}

int tk_jacobi_sweep(const tk_level* L, const double* b, const double* x_in, double* x_out,
                    double omega, void* stream) {
    TK_CHECK_ARG(b && x_out, "tk_jacobi_sweep: null vector");
    TK_CHECK_ARG(x_in != x_out, "tk_jacobi_sweep: x_out must not alias x_in");
    return level_op(L, 4, 4, b, x_in, x_out, omega, stream);
}

static bool dense_jacobi0_restrict_ok(const tk_level* L, double omega) {
    const bool whole = L->row0 == 0 && (L->row1 == 0 || L->row1 == L->n_steps + 1);
    return L->family == TK_FAMILY_DENSE && omega == 1.0 && whole && (L->n_steps % 2) == 0 &&
           L->n_steps >= 2 && L->n_u >= 1 && L->n_u <= TK_MAX_DENSE && L->n_z >= 1 &&
           L->n_z <= TK_MAX_DENSE;
}

// the u/mu-only pre-smoothing + folded prolongation (dense_rows_split) also run on
// a time slab cut at even rows
static bool dense_pair_ok(const tk_level* L, double omega) {
    const int r1 = L->row1 > 0 ? L->row1 : L->n_steps + 1;
    const bool slab = (L->row0 & 1) == 0 && (r1 == L->n_steps + 1 || (r1 & 1) == 0) &&
                      r1 - L->row0 >= 2;
    return L->family == TK_FAMILY_DENSE && omega == 1.0 && slab && (L->n_steps % 2) == 0 &&
           L->n_steps >= 2 && L->n_u >= 1 && L->n_u <= TK_MAX_DENSE && L->n_z >= 1 &&
           L->n_z <= TK_MAX_DENSE;
}

int32_t tk_jacobi0_restrict_ok(const tk_level* L, double omega) {
    if (check_level(L)) return 0;
    if (L->family == TK_FAMILY_DENSE) return dense_jacobi0_restrict_ok(L, omega) ? 1 : 0;
    return tri_jacobi0_restrict_ok(L, omega) ? 1 : 0;
}

int tk_jacobi0_restrict(const tk_level* L, const double* b, double omega, double* x_out, double* rc,
                        void* stream) {
    TK_CHECK_ARG(b && x_out && rc, "tk_jacobi0_restrict: null vector");
    const int e = check_level(L);
    if (e) return e;
    if (L->family == TK_FAMILY_DENSE) {
        if (!dense_jacobi0_restrict_ok(L, omega)) {
            set_error("tk_jacobi0_restrict: level not supported (whole level, even N, omega = 1)");
            return TK_ERR_UNSUPPORTED;
        }
        return dense_jacobi0_restrict(L, b, x_out, rc, as_stream(stream));
    }
    return tri_jacobi0_restrict_launch(L, b, omega, x_out, rc, as_stream(stream));
}

int32_t tk_jacobi_prolong_ok(const tk_level* L, double omega) {
    if (check_level(L)) return 0;
    if (L->family == TK_FAMILY_DENSE) return dense_pair_ok(L, omega) ? 1 : 0;
    return tri_jacobi_prolong_ok(L, omega) ? 1 : 0;
}

int tk_jacobi0_restrict_um(const tk_level* L, const double* b, double* x_um, double* rc,
                           void* stream) {
    TK_CHECK_ARG(b && x_um && rc, "tk_jacobi0_restrict_um: null vector");
    const int e = check_level(L);
    if (e) return e;
    if (!tk_jacobi_prolong_ok(L, 1.0)) {
        set_error("tk_jacobi0_restrict_um: level not supported (see tk_jacobi_prolong_ok)");
        return TK_ERR_UNSUPPORTED;
    }
    if (L->family == TK_FAMILY_DENSE)
        return dense_split(L, b, nullptr, x_um, nullptr, rc, 1, as_stream(stream));
    return tri_jacobi0_restrict_launch(L, b, 1.0, x_um, rc, as_stream(stream), 1);
}

int tk_jacobi_restrict(const tk_level* L, const double* b, const double* x_in, double* x_out,
                       double* rc, void* stream) {
    TK_CHECK_ARG(b && x_out && rc && x_in != x_out, "tk_jacobi_restrict: bad vectors");
    const int e = check_level(L);
    if (e) return e;
    if (!(L->family == TK_FAMILY_DENSE ? dense_pair_ok(L, 1.0) : tk_jacobi0_restrict_ok(L, 1.0) != 0)) {
        set_error("tk_jacobi_restrict: level not supported (see tk_jacobi0_restrict_ok)");
        return TK_ERR_UNSUPPORTED;
    }
    if (L->family == TK_FAMILY_DENSE)
        return dense_split(L, b, x_in, x_out, nullptr, rc, 0, as_stream(stream));
    return tri_jacobi_restrict_launch(L, b, x_in, x_out, rc, as_stream(stream));
}

int tk_jacobi_prolong(const tk_level* L, const double* b, const double* x, const double* ec,
                      double* x_out, void* stream) {
    TK_CHECK_ARG(b && x && ec && x_out && x != x_out && b != x_out, "tk_jacobi_prolong: bad vectors");
    const int e = check_level(L);
    if (e) return e;
    if (L->family == TK_FAMILY_DENSE) {
        if (!dense_jacobi0_restrict_ok(L, 1.0)) {
            set_error("tk_jacobi_prolong: level not supported (whole level, even N)");
            return TK_ERR_UNSUPPORTED;
        }
        return dense_split(L, b, x, x_out, ec, nullptr, 0, as_stream(stream));
    }
    return tri_jacobi_prolong_launch(L, b, x, ec, x_out, as_stream(stream));
}

int tk_jacobi_prolong_slab(const tk_level* L, const double* b, const double* x, const double* ec,
                           const double* chalo, double* x_out, void* stream) {
    TK_CHECK_ARG(b && x && ec && chalo && x_out && x != x_out && b != x_out,
                 "tk_jacobi_prolong_slab: bad vectors");
    const int e = check_level(L);
    if (e) return e;
    if (L->family == TK_FAMILY_DENSE) {
        if (!dense_pair_ok(L, 1.0)) {
            set_error("tk_jacobi_prolong_slab: level not supported (slab cut at even rows, even N)");
            return TK_ERR_UNSUPPORTED;
        }
        return dense_split(L, b, x, x_out, ec, nullptr, 0, as_stream(stream), chalo);
    }
    return tri_jacobi_prolong_launch(L, b, x, ec, x_out, as_stream(stream), chalo);
}

int tk_restrict_fix_slab(const tk_level* L, double* rc, void* stream) {
    TK_CHECK_ARG(rc, "tk_restrict_fix_slab: null vector");
    const int e = check_level(L);
    if (e) return e;
    return tri_restrict_fix_slab_launch(L, rc, as_stream(stream));
}

int tk_restrict_fix_slab_x(const tk_level* L, double* rc, int32_t phase, void* stream) {
    TK_CHECK_ARG(rc && (phase == 1 || phase == 2), "tk_restrict_fix_slab_x: bad arguments");
    const int e = check_level(L);
    if (e) return e;
    return tri_restrict_fix_slab_launch(L, rc, as_stream(stream), phase);
}

int tk_forward_subst(const tk_level* L, const double* r, double* delta, void* stream) {
    TK_CHECK_ARG(r && delta && r != delta, "tk_forward_subst: bad vectors");
    return level_op(L, 10, 10, r, nullptr, delta, 1.0, stream);
}

int tk_backward_subst(const tk_level* L, const double* r, double* delta, void* stream) {
    TK_CHECK_ARG(r && delta && r != delta, "tk_backward_subst: bad vectors");
    return level_op(L, 11, 11, r, nullptr, delta, 1.0, stream);
}

int tk_sgs_back_half(const tk_level* L, const double* w, double* d, void* stream) {
    TK_CHECK_ARG(w && d && w != d, "tk_sgs_back_half: bad vectors");
    int rc = check_level(L);
    if (rc) return rc;
    if (L->family != TK_FAMILY_TRI) {
        set_error("tk_sgs_back_half: TRI levels only (use apply_diag + backward_subst)");
        return TK_ERR_UNSUPPORTED;
    }
    return tri_launch(L, 14, w, nullptr, d, 1.0, as_stream(stream));
}

int64_t tk_subst_factor_len(const tk_level* L) {
    if (check_level(L)) return -1;
    return L->family == TK_FAMILY_DENSE ? dense_fac_len(L) : tri_fac_len(L);
}

int64_t tk_subst_scratch_len(const tk_level* L) {
    if (check_level(L)) return -1;
    return L->family == TK_FAMILY_DENSE ? dense_scratch_len(L) : tri_scratch_len(L);
}

int tk_subst_factor(const tk_level* L, void* stream) {
    return level_op(L, 12, 12, nullptr, nullptr, nullptr, 1.0, stream);
}

int32_t tk_chain_chunk_default(int32_t n_u, int32_t n_steps) {
    return tri_chain_chunk_default(n_u, n_steps);
}

int64_t tk_chain_prod_len(const tk_level* L) {
    if (check_level(L)) return -1;
    return L->family == TK_FAMILY_TRI ? tri_chain_prod_len(L) : 0;
}

int tk_chain_prod(const tk_level* L, void* stream) {
    int rc = check_level(L);
    if (rc) return rc;
    if (L->family != TK_FAMILY_TRI) {
        set_error("tk_chain_prod: only the TRI family chunks its chain");
        return TK_ERR_UNSUPPORTED;
    }
    return tri_launch(L, 13, nullptr, nullptr, nullptr, 1.0, as_stream(stream));
}

int32_t tk_tri_cut_nodes(int32_t n_u) { return n_u >= 1 ? tri_cut_nodes(n_u) : 0; }

int tk_tri_cut_indices(int32_t n_u, int32_t* out) {
    TK_CHECK_ARG(n_u >= 1 && out, "tk_tri_cut_indices: bad arguments");
    const int c = tri_cut_level(n_u), a = tri_cut_nodes(n_u);
    for (int m = 0; m < a; ++m) out[m] = ((m + 1) << c) - 1;
    return TK_OK;
}

int tk_restrict(int32_t n_fine, int32_t n_u, int32_t n_z, const double* xf, double* xc,
                void* stream) {
    TK_CHECK_ARG(xf && xc && n_fine >= 2 && n_fine % 2 == 0 && n_u >= 1 && n_z >= 1,
                 "tk_restrict: bad arguments (n_fine must be even)");
    return transfer_launch(1, n_fine, n_u, n_z, 0, 0, xf, nullptr, nullptr, xc,
                           as_stream(stream));
}

int tk_prolong_add(int32_t n_fine, int32_t n_u, int32_t n_z, const double* xc, double* xf,
                   void* stream) {
    TK_CHECK_ARG(xf && xc && n_fine >= 2 && n_fine % 2 == 0 && n_u >= 1 && n_z >= 1,
                 "tk_prolong_add: bad arguments (n_fine must be even)");
    return transfer_launch(0, n_fine, n_u, n_z, 0, 0, xc, nullptr, nullptr, xf,
                           as_stream(stream));
}

int tk_restrict_slab(int32_t n_fine, int32_t n_u, int32_t n_z, int32_t row0, int32_t row1,
                     const double* xf, double* xc, void* stream) {
    TK_CHECK_ARG(xf && xc && n_fine >= 2 && n_fine % 2 == 0 && n_u >= 1 && n_z >= 1,
                 "tk_restrict_slab: bad arguments (n_fine must be even)");
    return transfer_launch(1, n_fine, n_u, n_z, row0, row1, xf, nullptr, nullptr, xc,
                           as_stream(stream));
}

int tk_prolong_add_slab(int32_t n_fine, int32_t n_u, int32_t n_z, int32_t row0, int32_t row1,
                        const double* xc, const double* halo_prev_ul,
                        const double* halo_next_vm, double* xf, void* stream) {
    TK_CHECK_ARG(xf && xc && n_fine >= 2 && n_fine % 2 == 0 && n_u >= 1 && n_z >= 1,
                 "tk_prolong_add_slab: bad arguments (n_fine must be even)");
    return transfer_launch(0, n_fine, n_u, n_z, row0, row1, xc, halo_prev_ul, halo_next_vm, xf,
                           as_stream(stream));
}

int tk_residual_restrict(const tk_level* L, const double* b, const double* x, double* rc,
                         double* work, void* stream) {
    TK_CHECK_ARG(b && x && rc && work, "tk_residual_restrict: null vector");
    {
        const int e = check_level(L);
        if (e) return e;
    }
    if (L->family == TK_FAMILY_TRI)   // fused: the fine residual never reaches HBM
        return tri_resrestrict_launch(L, b, x, rc, as_stream(stream));
    int rcode = level_op(L, 2, 2, b, x, work, 1.0, stream);
    if (rcode) return rcode;
    return transfer_launch(1, L->n_steps, L->n_u, L->n_z, L->row0, L->row1, work, nullptr,
                           nullptr, rc, as_stream(stream));
}

int tk_residual_restrict_jacobi0(const tk_level* L, const double* b, const double* x,
                                 double omega, double* rc, void* stream) {
    TK_CHECK_ARG(x && rc && (b || omega == 1.0), "tk_residual_restrict_jacobi0: null vector");
    int e = check_level(L);
    if (e) return e;
    if (L->n_steps & 1) {
        set_error("tk_residual_restrict_jacobi0: odd step count");
        return TK_ERR_ARG;
    }
    return restrict_jacobi0_launch(L->n_steps, L->n_u, L->n_z, L->row0, L->row1, b, x, L->halo_u,
                                   L->halo_mu, omega, rc, as_stream(stream));
}

int64_t tk_reduce_work_len(void) { return reduce_work_len(); }

int tk_dot(int64_t n, const double* x, const double* y, double* out, double* work,
           void* stream) {
    TK_CHECK_ARG(x && y && out && work && n >= 0, "tk_dot: bad arguments");
    return dot_launch(n, x, y, out, work, 0, as_stream(stream));
}

int tk_nrm2(int64_t n, const double* x, double* out, double* work, void* stream) {
    TK_CHECK_ARG(x && out && work && n >= 0, "tk_nrm2: bad arguments");
    return dot_launch(n, x, x, out, work, 1, as_stream(stream));
}

int tk_axpy(int64_t n, double a, const double* x, double* y, void* stream) {
    TK_CHECK_ARG(x && y, "tk_axpy: null vector");
    return vec_launch(0, n, a, x, y, as_stream(stream));
}

int tk_scale_into(int64_t n, double a, const double* x, double* y, void* stream) {
    TK_CHECK_ARG(x && y, "tk_scale_into: null vector");
    return vec_launch(1, n, a, x, y, as_stream(stream));
}

int tk_axpy_dev(int64_t n, const double* a, double sign, const double* x, double* y,
                void* stream) {
    TK_CHECK_ARG(a && x && y && n >= 0, "tk_axpy_dev: bad arguments");
    return axpy_dev_launch(n, a, sign, x, y, as_stream(stream));
}

int tk_sqrt_div(int64_t n, const double* sq, double* nrm, const double* x, double* y,
                void* stream) {
    TK_CHECK_ARG(sq && n >= 0 && (!y || x), "tk_sqrt_div: bad arguments");
    // every CTA reads sq[0] while one thread writes nrm[0]: in place would race
    TK_CHECK_ARG(nrm != sq, "tk_sqrt_div: nrm must not alias sq");
    return sqrt_div_launch(n, sq, nrm, x, y, as_stream(stream));
}

int tk_rsub(int64_t n, const double* b, double* y, void* stream) {
    TK_CHECK_ARG(b && y, "tk_rsub: null vector");
    return vec_launch(2, n, 0.0, b, y, as_stream(stream));
}

int tk_copy_kernel(int64_t n, const double* src, double* dst, void* stream) {
    TK_CHECK_ARG(src && dst && n >= 0, "tk_copy_kernel: bad arguments");
    if (n == 0) return TK_OK;
    return copy_small_launch(n, src, dst, as_stream(stream));
}

int tk_host_alloc_mapped(int64_t bytes, void** host, void** dptr) {
    TK_CHECK_ARG(bytes > 0 && host && dptr, "tk_host_alloc_mapped: bad arguments");
    int rc = cuda_status(cudaHostAlloc(host, (size_t)bytes, cudaHostAllocMapped | cudaHostAllocPortable),
                         "cudaHostAlloc");
    if (rc) return rc;
    return cuda_status(cudaHostGetDevicePointer(dptr, *host, 0), "cudaHostGetDevicePointer");
}

int tk_host_free(void* host) { return cuda_status(cudaFreeHost(host), "cudaFreeHost"); }

int tk_host_device_ptr(void* host, void** dptr) {
    TK_CHECK_ARG(host && dptr, "tk_host_device_ptr: bad arguments");
    return cuda_status(cudaHostGetDevicePointer(dptr, host, 0), "cudaHostGetDevicePointer");
}

int tk_arnoldi_mgs(int64_t n, int32_t j, double* V, int64_t ld, double* w, double* h,
                   double* work, void* stream) {
    TK_CHECK_ARG(V && w && h && work && n >= 0 && j >= 0 && ld >= n,
                 "tk_arnoldi_mgs: bad arguments");
    return arnoldi_launch(n, j, V, ld, w, h, work, as_stream(stream));
}

int32_t tk_arnoldi_supported(void) { return arnoldi_supported() ? 1 : 0; }

int tk_l2_persist_reset(void) { return l2_persist_reset(); }
int tk_l2_persist_allow(int32_t on) { return l2_persist_allow(on); }

int tk_gemv_t_add(int64_t n, int32_t k, const double* V, int64_t ld, const double* c, double* x,
                  void* stream) {
    TK_CHECK_ARG(V && c && x && k >= 0 && ld >= n, "tk_gemv_t_add: bad arguments");
    if (k == 0) return TK_OK;
    return gemv_t_add_launch(n, k, V, ld, c, x, as_stream(stream));
}

int tk_stage_vanderpol(int32_t n_steps, double dt, double theta, double mu, int32_t n_controls,
                       const double* u0, const double* u, const double* v, const double* z,
                       double* K, double* C, double* B, void* stream) {
    TK_CHECK_ARG(n_steps >= 1 && (n_controls == 1 || n_controls == 2) && u0 && u && v && K && C &&
                     B,
                 "tk_stage_vanderpol: bad arguments");
    return stage_vdp_launch(n_steps, dt, theta, mu, n_controls, u0, u, v, z, K, C, B,
                            as_stream(stream));
}

int tk_stage_burgers(int32_t n_steps, int32_t n_u, double dt, double theta, double nu,
                     const double* u0, const double* u, const double* v, double* K, double* C,
                     void* stream) {
    TK_CHECK_ARG(n_steps >= 1 && n_u >= 2 && u0 && u && v && K && C,
                 "tk_stage_burgers: bad arguments");
    return stage_burgers_launch(n_steps, n_u, dt, theta, nu, u0, u, v, K, C, as_stream(stream));
}

int tk_check_k(const tk_level* L, double pivot_floor, int32_t* bad, void* stream) {
    int rc = check_level(L);
    if (rc != TK_OK) return rc;
    TK_CHECK_ARG(bad && pivot_floor >= 0.0, "tk_check_k: bad arguments");
    return check_k_launch(L, pivot_floor, bad, as_stream(stream));
}

int tk_check_blocks(const tk_level* L, double pivot_floor, int32_t* bad, void* stream) {
    int rc = check_level(L);
    if (rc != TK_OK) return rc;
    TK_CHECK_ARG(bad && pivot_floor >= 0.0, "tk_check_blocks: bad arguments");
    if (L->family != TK_FAMILY_DENSE || L->row0 != 0 || L->row1 != 0) {
        set_error("tk_check_blocks: whole DENSE levels only");
        return TK_ERR_UNSUPPORTED;
    }
    return check_blocks_launch(L, pivot_floor, bad, as_stream(stream));
}

}  // extern "C"
