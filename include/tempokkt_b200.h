/*
 * tempokkt_b200.h -- C-ABI of the B200-native hot path of the
 * multigrid-in-time KKT preconditioner (arXiv 2405.04808).
 *
 * Every entry point takes plain pointers and sizes (device pointers for
 * vectors and stage data, a cudaStream_t passed as void*), returns an int
 * status (TK_OK == 0) and never allocates on the hot path.  Each function
 * names the reference interface it replaces (file:line inside
 * /root/reference/pkg/src/tempokkt/).  INTEGRATION.md shows the ctypes
 * binding the reference would add.
 *
 * Vector layout: exactly the reference's time-clustered ordering
 * (kkt.py:6-16, KktLayout kkt.py:127-191):
 *   block 0       (u_1, z_1, lam_1)                      size 2nu+nz
 *   block i=1..N-1 (v_i, u_{i+1}, z_{i+1}, mu_i, lam_{i+1}) size 4nu+nz
 *   block N       (v_N, mu_N)                             size 2nu
 * so a device vector is bit-compatible with the reference's numpy vector.
 */
#ifndef TEMPOKKT_B200_H
#define TEMPOKKT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TK_OK 0
#define TK_ERR_ARG 1          /* bad sizes / null pointers  (errors.py:8 DimensionMismatch) */
#define TK_ERR_CUDA 2         /* CUDA runtime error                                        */
#define TK_ERR_UNSUPPORTED 3  /* structure not supported by the kernels                    */
#define TK_ERR_NEWTON 4       /* forward Newton failed      (errors.py:40 NewtonDivergence) */

#define TK_FAMILY_DENSE 0     /* small dense stage blocks (van der Pol): nu<=4, nz<=4       */
#define TK_FAMILY_TRI 1       /* tridiagonal-in-space stage blocks (1D FE Burgers), nz==nu  */

#define TK_MAX_DENSE 4
/* DENSE levels beyond TK_MAX_DENSE (general dense stage blocks, e.g. the
 * reference's heat-Neumann problem): one warp per block row, the local saddle
 * system by pivoted elimination in shared memory; n_u <= 40, n_z <= 8.  The
 * fused V(1,1) kernels and the substitution factor records cover the small
 * sizes only (tk_jacobi0_restrict_ok / tk_jacobi_prolong_ok return 0; no
 * tk_subst_factor: the substitutions run as one serial kernel). */
#define TK_MAX_DENSE_GENERAL 40

/*
 * One level of the operator ladder (replaces BlockTriKKT + DiagonalSolver,
 * kkt.py:194-389, built per level by multigrid.py:190-242).
 *
 * Stage data are the reference's StageBlocks (kkt.py:53-80):
 *   DENSE: K,C [N][nu][nu], B [N][nu][nz], row-major (same as numpy).
 *   TRI:   K,C [N][3][nu] as (sub, diag, sup) diagonals; sub[0]=sup[nu-1]=0.
 *          B is not stored: the family requires B_i = kappa * Qz (checked at
 *          setup), which holds for the reference's Burgers (F_z = M,
 *          w_control = alpha*M => kappa = 1/alpha).
 * Weights (timedisc.py:194-206) are time-constant except the terminal stage:
 *   Qm = q_u[i] = q_v[i] for i < N-1, Ql = q_u[N-1] = q_v[N-1], Qz = q_z[i].
 *   DENSE: [nu][nu] / [nz][nz] plus their inverses (Qm_inv, Ql_inv, Qz_inv).
 *   TRI:   [3][nu] diagonals; qz_cr = [3][nu] scalar cyclic-reduction
 *          coefficients of Qz from tk_cr_scalar_factor().
 */
typedef struct tk_level {
    int32_t family;
    int32_t n_steps;
    int32_t n_u;
    int32_t n_z;
    const double* K;
    const double* C;
    const double* B;
    const double* Qm;
    const double* Ql;
    const double* Qz;
    const double* Qm_inv;
    const double* Ql_inv;
    const double* Qz_inv;
    double kappa;
    const double* qz_cr;
    /* Optional Gauss-Seidel acceleration data (see tk_subst_factor):
     * fac     precomputed local-solve factors   (tk_subst_factor_len doubles)
     * scratch coupling-chain buffer             (tk_subst_scratch_len doubles)
     * When both are set, tk_forward_subst / tk_backward_subst run as
     * parallel solve -> serial n_u-vector chain -> parallel solve. */
    double* fac;
    double* scratch;
    /* Time slab (multi-GPU sharding).  The level handles global block rows
     * [row0, row1) (row1 == 0 means n_steps+1, i.e. the whole level); every
     * vector argument is then the LOCAL slice starting at the global offset of
     * row0, and K, C, B hold stages [row0, min(row1, n_steps)).  The continuity
     * couplings across the slab edges come from two n_u halo buffers:
     *   halo_u  = u-segment of global row row0-1   (required if row0 > 0)
     *   halo_mu = mu-segment of global row row1    (required if row1 <= n_steps)
     * refreshed by the caller's neighbour exchange before each call.  The
     * serial-in-time substitutions require the whole level (no slab). */
    int32_t row0;
    int32_t row1;
    const double* halo_u;
    const double* halo_mu;
    /* TRI: transposed dense inverse of the scalar Q_z system reduced to the
     * cyclic-reduction cut level (tk_tri_cut_nodes(n_u)^2 doubles, i.e. the
     * (active, active) block of Q_z^{-1}).  Required by every TRI local
     * solve; with factor records in L->fac, D^{-1} runs rhs-only. */
    const double* qz_w;
    /* TRI: time-chunked coupling chain (see tk_chain_prod).  With chain_chunk
     * = Lc > 0 and chain_prod filled by tk_chain_prod, the serial n_u-vector
     * chain of the substitutions runs as: all chunks of Lc intervals in
     * parallel from a zero start -> a short serial carry over the chunk ends
     * with the precomputed chunk propagators -> all chunks again from their
     * true start.  chain_chunk = 0: one serial chain. */
    double* chain_prod;
    int32_t chain_chunk;
    /* TK_FLAG_ONTHEFLY: TRI local solves (Jacobi, diagonal solve, the
     * parallel passes of the substitutions) refactor on the fly even when
     * L->fac holds factor records.  By default records drive them only where
     * the partitioned on-the-fly solve cannot run (n_u > 2048);
     * TK_FLAG_RECROWS forces the record-based kernels whenever records exist. */
    int32_t flags;
} tk_level;

#define TK_FLAG_ONTHEFLY 1
#define TK_FLAG_RECROWS 2
/* TK_FLAG_TOEPLITZ_W: the TRI weights Qm, Ql, Qz have constant diagonals
 * (sub[1:] == sup[:-1] == s, diag == d; uniform P1 mass matrices), set by the
 * host after checking; the partitioned row kernels then read one scalar per
 * diagonal instead of per-node values (same values, bitwise same results). */
#define TK_FLAG_TOEPLITZ_W 4

/* --- library ------------------------------------------------------------ */
const char* tk_version(void);
const char* tk_last_error(void);
/* dim = N*(4nu+nz) (kkt.py:141). */
int64_t tk_kkt_dim(int32_t n_steps, int32_t n_u, int32_t n_z);
/* Bytes of dynamic shared memory the TRI kernels need for n_u (0 = unsupported). */
int64_t tk_tri_smem_bytes(int32_t n_u);

/* --- the operator (kkt.py) ---------------------------------------------- */
/* y = A x                        replaces BlockTriKKT.apply        kkt.py:228 */
int tk_kkt_apply(const tk_level* L, const double* x, double* y, void* stream);
/* r = b - A x                    replaces `b - a.apply(x)`   smoothers.py:74, multigrid.py:288 */
int tk_kkt_residual(const tk_level* L, const double* b, const double* x, double* r,
                    void* stream);
/* y = D x (no continuity couplings) replaces split_parts' D        kkt.py:400 and smoothers.py:142-151 */
int tk_kkt_apply_diag(const tk_level* L, const double* x, double* y, void* stream);
/* y = D^{-1} r  (all block rows in parallel) replaces DiagonalSolver.solve_all kkt.py:377 */
int tk_diag_solve(const tk_level* L, const double* r, double* y, void* stream);

/* --- smoothers (smoothers.py) --------------------------------------------- */
/* One block-Jacobi sweep x_out = x_in + omega*D^{-1}(b - A x_in); x_in may be NULL
 * (zero initial guess).  x_out must not alias x_in.  replaces jacobi_apply smoothers.py:61 */
int tk_jacobi_sweep(const tk_level* L, const double* b, const double* x_in, double* x_out,
                    double omega, void* stream);
/* (D - L) delta = r, serial in time   replaces _forward_subst  smoothers.py:79 */
int tk_forward_subst(const tk_level* L, const double* r, double* delta, void* stream);
/* (D - U) delta = r, serial in time   replaces _backward_subst smoothers.py:95 */
int tk_backward_subst(const tk_level* L, const double* r, double* delta, void* stream);
/* d = (D - U)^{-1} D w, the second half of the symmetric Gauss-Seidel
 * (smoothers.py:130-152: `(D-U)^{-1} D (D-L)^{-1} r` with w = (D-L)^{-1} r).
 * Pass 1 of the backward substitution would form D^{-1} (D w) = w, so the
 * coupling chain starts from w and the parallel pass solves a zero rhs on top
 * of w.  TRI levels with factor records (after tk_subst_factor); other levels
 * return TK_ERR_UNSUPPORTED. */
int tk_sgs_back_half(const tk_level* L, const double* w, double* d, void* stream);
/* Sizes (in doubles) of L->fac and L->scratch, and the one-off factorisation
 * filling L->fac (TRI: per-interval cyclic-reduction factors of the (u,lam)
 * system + C_i; DENSE: the n_u x n_u chain matrices P_u D_i^{-1} E_mu and
 * P_mu D_i^{-1} E_u).  Built once per level (kkt.py:338 DiagonalSolver). */
int64_t tk_subst_factor_len(const tk_level* L);
int64_t tk_subst_scratch_len(const tk_level* L);
int tk_subst_factor(const tk_level* L, void* stream);
/* TRI: cut level / active-node count of the record-based local solves, and
 * the node indices (0-based) of the active nodes (host memory, out[cut_nodes]). */
int32_t tk_tri_cut_nodes(int32_t n_u);
int tk_tri_cut_indices(int32_t n_u, int32_t* out);
/* TRI chunked chain: default chunk length for (n_u, n_steps) (0 = keep the
 * chain serial), the size in doubles of L->chain_prod for L->chain_chunk, and
 * the one-off computation of the chunk propagators Pi_c = T_hi-1 ... T_lo
 * (T_i: u_{i-1} -> u_i of the homogeneous forward chain; the backward chain
 * uses Pi_c^T since the local (u,lam) systems are symmetric).  Needs L->fac
 * (tk_subst_factor) first. */
int32_t tk_chain_chunk_default(int32_t n_u, int32_t n_steps);
int64_t tk_chain_prod_len(const tk_level* L);
int tk_chain_prod(const tk_level* L, void* stream);

/* --- transfers (multigrid.py:104-132) ------------------------------------- */
/* xc = R xf  (injection for u,v,lam,mu; 2-interval average for z)    restrict_kkt multigrid.py:104 */
int tk_restrict(int32_t n_fine, int32_t n_u, int32_t n_z, const double* xf, double* xc,
                void* stream);
/* xf += P xc (linear interpolation / piecewise-constant copy)  prolong_kkt + `x + t.prolong_kkt(e)`
 * multigrid.py:115 and :297 */
int tk_prolong_add(int32_t n_fine, int32_t n_u, int32_t n_z, const double* xc, double* xf,
                   void* stream);
/* Slab versions for the time-sharded hierarchy: [row0, row1) are FINE block
 * rows (row0 even; row1 even or n_fine+1), the coarse slice covers coarse rows
 * [row0/2, row1/2) (or through n_fine/2 for the last slab).  Restriction is
 * slab-local; prolongation needs the previous slab's last coarse (u, lam)
 * segments (halo_prev_ul, 2 n_u) and the next slab's first coarse (v, mu)
 * segments (halo_next_vm, 2 n_u).  tk_restrict / tk_prolong_add are the
 * whole-level special case. */
int tk_restrict_slab(int32_t n_fine, int32_t n_u, int32_t n_z, int32_t row0, int32_t row1,
                     const double* xf, double* xc, void* stream);
int tk_prolong_add_slab(int32_t n_fine, int32_t n_u, int32_t n_z, int32_t row0, int32_t row1,
                        const double* xc, const double* halo_prev_ul,
                        const double* halo_next_vm, double* xf, void* stream);
/* rc = R (b - A x)  (work: fine-sized scratch; honours the level's slab)  multigrid.py:288 */
/* rc = R (b - A x) when x is ONE block-Jacobi sweep from zero (x = omega
 * D^{-1} b, the V-cycle pre-smoothing with sweeps = 1, multigrid.py:284-288):
 * D x = omega b, so b - A x = (1 - omega) b - (L + U) x reduces to the
 * continuity couplings (r_mu(t) -= u_t, r_u(t) -= mu_t) -- b is not read for
 * omega == 1 and x only at the injected u/mu segments.  Time slabs read the
 * coupling partners outside the slab from L->halo_u / L->halo_mu. */
int tk_residual_restrict_jacobi0(const tk_level* L, const double* b, const double* x,
                                 double omega, double* rc, void* stream);
/* The V-cycle's zero-start pre-smoothing sweep and its restricted residual
 * in ONE pass (multigrid.py:284-288 with one sweep from zero): x_out =
 * D^{-1} b (tk_jacobi_sweep with x_in = NULL, omega = 1) and rc exactly as
 * tk_residual_restrict_jacobi0(L, b, x_out, 1, rc).  DENSE levels and TRI
 * levels of the partitioned row solve; whole level, even N, omega == 1:
 * check tk_jacobi0_restrict_ok(), else TK_ERR_UNSUPPORTED. */
int32_t tk_jacobi0_restrict_ok(const tk_level* L, double omega);
int tk_jacobi0_restrict(const tk_level* L, const double* b, double omega, double* x_out,
                        double* rc, void* stream);
int tk_residual_restrict(const tk_level* L, const double* b, const double* x, double* rc,
                         double* work, void* stream);
/* V(1,1) with omega = 1 (multigrid.py:284-299, one sweep each side): the
 * post-smoothing sweep x + D^{-1}(b - A x) equals D^{-1}(b + (L + U) x), and
 * (L + U) x reads only the continuity couplings u_{i-1}, mu_{i+1} of x.  So
 * the prolongation x + P ec (multigrid.py:115-132, :297) folds into the sweep:
 *   x_out = D^{-1}(b + (L + U)(x + P ec))
 * reads the u and mu segments of x and of the coarse correction ec and never
 * forms x + P ec in HBM (same arithmetic per element as tk_prolong_add then
 * tk_jacobi_sweep with omega = 1).  tk_jacobi0_restrict_um is the matching
 * pre-smoothing: tk_jacobi0_restrict storing ONLY the u and mu segments of
 * its x (the other segments of x_um are left untouched), which is all the
 * fused post-smoothing reads.  DENSE levels (n_u, n_z <= 4) and TRI levels of
 * the partitioned rows (4 < n_u <= 2048); whole level, even N: check
 * tk_jacobi_prolong_ok(), else TK_ERR_UNSUPPORTED. */
int32_t tk_jacobi_prolong_ok(const tk_level* L, double omega);
/* One omega = 1 sweep from x_in (NULL: from zero) that also writes its
 * restricted residual rc = R (b - A x_out) (multigrid.py:285-288 with any
 * number of sweeps: the LAST pre-smoothing sweep).  After an omega = 1 sweep
 * D x_out = b + (L + U) x_in, hence b - A x_out = (L + U)(x_out - x_in): only
 * the continuity couplings of the update, which the sweep has in registers.
 * Where tk_jacobi0_restrict_ok(L, 1) holds. */
int tk_jacobi_restrict(const tk_level* L, const double* b, const double* x_in, double* x_out,
                       double* rc, void* stream);
int tk_jacobi0_restrict_um(const tk_level* L, const double* b, double* x_um, double* rc,
                           void* stream);
/* The fused V(1,1) pair on a TIME SLAB (both families; L->row0 even, L->row1 even
 * or n_steps+1; tk_jacobi0_restrict_ok / tk_jacobi_prolong_ok say yes for such
 * slabs too).  tk_jacobi0_restrict(_um) / tk_jacobi_restrict write the coarse
 * entries (local coarse slice, as tk_restrict_slab) their own rows feed; the
 * slab's first coarse mu comes from the previous slab's last row and its last
 * coarse u from the next slab's first row: after the halo exchange of the
 * iterate (L->halo_u / L->halo_mu, needed by the post-smoothing anyway)
 * tk_restrict_fix_slab writes those two segments (zero-start sweeps:
 * rc = -halo).  tk_jacobi_prolong_slab is tk_jacobi_prolong with the coarse
 * segments outside the slab taken from chalo = [previous slab's last coarse
 * (u, lam) | next slab's first coarse (v, mu)] (4 n_u doubles; the two halves
 * are tk_prolong_add_slab's halo_prev_ul / halo_next_vm).
 * Reference: multigrid.py:104-132, :285-299 on one time slab. */
int tk_restrict_fix_slab(const tk_level* L, double* rc, void* stream);
/* The same two segments after tk_jacobi_restrict from a NON-zero iterate x
 * (several sweeps): they are (x - y) of the neighbours' rows, so phase 1
 * (halos = those of x, i.e. before the exchange of y) stores +halo and phase 2
 * (halos = those of y) subtracts the halo. */
int tk_restrict_fix_slab_x(const tk_level* L, double* rc, int32_t phase, void* stream);
int tk_jacobi_prolong_slab(const tk_level* L, const double* b, const double* x, const double* ec,
                           const double* chalo, double* x_out, void* stream);
int tk_jacobi_prolong(const tk_level* L, const double* b, const double* x, const double* ec,
                      double* x_out, void* stream);

/* --- Krylov vector kernels (krylov.py:77-191) ----------------------------- */
/* Deterministic reductions: fixed grid, fixed order.  `out` is a device scalar.
 * `work` is a device buffer of at least tk_reduce_work_len() doubles. */
int64_t tk_reduce_work_len(void);
int tk_dot(int64_t n, const double* x, const double* y, double* out, double* work, void* stream);
int tk_nrm2(int64_t n, const double* x, double* out, double* work, void* stream);
/* y += a*x;  y = a*x (scal into) ; x *= a */
int tk_axpy(int64_t n, double a, const double* x, double* y, void* stream);
int tk_scale_into(int64_t n, double a, const double* x, double* y, void* stream);
/* y = b - y  (used for r = b - A x when A x is already in y) */
int tk_rsub(int64_t n, const double* b, double* y, void* stream);
/* y += sign * a[0] * x with the scalar a in device memory (the sharded MGS:
 * `w -= h_i V_i` with h_i an allreduced dot that stays on the device). */
int tk_axpy_dev(int64_t n, const double* a, double sign, const double* x, double* y,
                void* stream);
/* nrm[0] = sqrt(sq[0]) (nrm may be NULL, must not alias sq) and, when it is nonzero and y is
 * given, y = x / nrm[0] (krylov.py:150-163 `hj1 = norm2(w)`, `V[j+1] = w / hj1`
 * with the squared norm allreduced on the device). */
int tk_sqrt_div(int64_t n, const double* sq, double* nrm, const double* x, double* y,
                void* stream);
/* x += V^T c: V is k rows of length n with leading dimension ld; c on device */
int tk_gemv_t_add(int64_t n, int32_t k, const double* V, int64_t ld, const double* c,
                  double* x, void* stream);

/* dst = src (n doubles) by a kernel, not a copy engine: with src or dst in
 * mapped pinned host memory (tk_host_device_ptr) the Krylov scalars cross
 * PCIe without queueing behind bulk host<->device copies of other streams. */
int tk_copy_kernel(int64_t n, const double* src, double* dst, void* stream);
/* Mapped pinned host memory (cudaHostAllocMapped): host and device addresses. */
int tk_host_alloc_mapped(int64_t bytes, void** host, void** dptr);
int tk_host_free(void* host);
/* Device address of pinned (cudaHostAlloc'd / torch pin_memory) host memory. */
int tk_host_device_ptr(void* host, void** dptr);

/* One modified Gram-Schmidt Arnoldi step, replacing the inner loop of
 * krylov.py:77-191 (`for i in range(j+1): h = dot(V_i, w); w -= h V_i`,
 * `hj1 = norm2(w)`, `V_{j+1} = w / hj1`) by ONE cooperative launch with a grid
 * barrier per basis vector.  V: rows 0..j+1 of length n, leading dimension
 * ld; w is updated in place; h (device, >= j+2 doubles) receives
 * h_0..h_j, h_{j+1}; V_{j+1} is written when h_{j+1} != 0.  Bitwise equal to
 * the tk_dot / tk_axpy / tk_nrm2 / tk_scale_into sequence. */
int tk_arnoldi_mgs(int64_t n, int32_t j, double* V, int64_t ld, double* w, double* h,
                   double* work, void* stream);
/* For 16 MB <= n*8 <= 192 MB (and at most twice the device's persisting
 * carve-out), tk_arnoldi_mgs marks w L2-persisting (access-policy window;
 * the carve-out is set to the device maximum on first use;
 * TK_ARNOLDI_PERSIST=0 disables it).  tk_l2_persist_reset() returns those
 * lines to normal status and gives the carve-out back (while it is set every
 * other kernel runs in the remaining L2 only); call it after synchronising,
 * at the end of a solve.  tk_l2_persist_allow(0) keeps nested solves (the
 * coarse GMRES inside an outer FGMRES) from claiming the window. */
int tk_l2_persist_reset(void);
int tk_l2_persist_allow(int32_t on);
/* 1 when tk_arnoldi_mgs / tk_gm_arnoldi can run on the current device: their
 * fixed cooperative grid (592 CTAs of 256 threads) must be co-resident, which
 * a MIG slice or an SM-limited MPS client may not allow.  When 0 they return
 * TK_ERR_UNSUPPORTED and the host runs the unfused tk_dot / tk_axpy / tk_nrm2
 * / tk_scale_into sequence (same reductions, bitwise equal). */
int32_t tk_arnoldi_supported(void);

/* --- CUDA-graph V-cycle with a device-side coarse GMRES ------------------- */
/* Replaces the host-driven loop of multigrid.py:245-260 (coarse_solve ->
 * krylov.py:77-191 gmres from x0 = 0, SGS right preconditioner) inside a
 * captured V-cycle (multigrid.py:269-301) so that a cycle replays as ONE
 * graph launch with no host round trip.  Capture runs on a non-default
 * stream; the coarse Arnoldi loop is a WHILE conditional node whose
 * condition the Givens kernel sets (cudaGraphSetConditional). */
int tk_graph_capture_begin(void* stream);
int tk_graph_cond_create(void* stream, uint64_t* handle);
int tk_graph_while_begin(void* stream, void* body_stream, uint64_t handle);
int tk_graph_while_end(void* body_stream);
int tk_graph_capture_end(void* stream, void** exec);
int tk_graph_launch(void* exec, void* stream);
int tk_graph_destroy(void* exec);
/* Device GMRES state for a basis of `cap` columns (header, H, g, cs, sn, y). */
int64_t tk_gm_state_len(int32_t cap);
/* beta = ||b||, target = rel_tol*beta, g_0 = beta, V_0 = vj = b/beta; the
 * condition is set to 0 (skip the loop) when the host path must take over. */
int tk_gm_begin(int64_t n, const double* b, double* V, int64_t ld, double* vj, double* state,
                int32_t cap, double rel_tol, int32_t max_iters, uint64_t handle, double* work,
                void* stream);
/* MGS step j (j read from the state) with w = A M^{-1} v_j; V_{j+1} also to vj. */
int tk_gm_arnoldi(int64_t n, double* V, int64_t ld, double* w, double* state, int32_t cap,
                  double* vj, double* work, void* stream);
/* Z[j] = z with j read from the state (before tk_gm_arnoldi advances it): the
 * preconditioned directions z_j = M^{-1} v_j of the loop are kept, so that the
 * solution of the cycle is x = Z y (tk_gm_combine on Z) instead of
 * M^{-1}(V y) -- the same vector for the fixed linear M^{-1} of the coarse
 * solve (SGS), without the extra preconditioner application of
 * krylov.py:165-176. */
int tk_gm_storez(int64_t n, const double* z, double* Z, int64_t ldz, const double* state,
                 int32_t cap, void* stream);
/* Givens update + stopping tests of krylov.py; sets the loop condition. */
int tk_gm_givens(double* state, int32_t cap, uint64_t handle, void* stream);
/* y = H^{-1} g, vy = V^T y. */
int tk_gm_combine(int64_t n, const double* V, int64_t ld, double* state, int32_t cap,
                  double* vy, void* stream);
/* r (= A x on entry) <- b - A x; ||r||, ||x||; res[0] = 1 when the host path
 * must redo the solve (restart, breakdown, non-finite, basis overflow),
 * res[1] = iterations.  res may be mapped host memory. */
int tk_gm_finish(int64_t n, const double* b, double* r, const double* x, double* state,
                 int32_t cap, int32_t* res, double* work, void* stream);

/* --- setup: stage linearisation on the device (timedisc.py:133, kkt.py:100) - */
/* van der Pol: K,C,B at (v_{i-1}, u_i, z_i), v_{-1} = u0.  n_controls in {1,2}. */
int tk_stage_vanderpol(int32_t n_steps, double dt, double theta, double mu, int32_t n_controls,
                       const double* u0, const double* u, const double* v, const double* z,
                       double* K, double* C, double* B, void* stream);
/* Burgers (problems.py:149): TRI diagonals of K, C at (v_{i-1}, u_i, z_i). */
int tk_stage_burgers(int32_t n_steps, int32_t n_u, double dt, double theta, double nu,
                     const double* u0, const double* u, const double* v, double* K, double* C,
                     void* stream);

/* --- setup: singularity checks (kkt.py:323-389, 496-543) ------------------- */
/* bad[s] = 1 when stage K_s fails the K half of Theorem 1 (check_theorem1
 * kkt.py:530-543): partial-pivoting LU (linalg.lu_factor linalg.py:75-103)
 * meets a pivot below pivot_floor*max|K_s| (reference PIVOT_FLOOR = 1e-14,
 * linalg.py:38) or K_s holds a non-finite entry.  One flag per local stage
 * of the level (slab: stages [row0, min(row1, N))).  The weight (SPD) half of
 * the theorem is checked by the host on the time-constant weights. */
int tk_check_k(const tk_level* L, double pivot_floor, int32_t* bad, void* stream);
/* bad[i] = 1 (i = 0..N) when the diagonal block of block row i, assembled as
 * assemble_kkt (kkt.py:279-320), fails the same partial-pivoting LU test --
 * where DiagonalSolver (kkt.py:347-368) raises SingularBlock(i).  Whole DENSE
 * levels (TRI blocks are quasi-definite once the weights are SPD, which the
 * host checks); TK_ERR_UNSUPPORTED otherwise. */
int tk_check_blocks(const tk_level* L, double pivot_floor, int32_t* bad, void* stream);

/* --- setup: host routines (CPU) ------------------------------------------- */
/* theta-method forward march with Newton (timedisc.py:152-191), host memory. */
int tk_forward_vanderpol_host(int32_t n_steps, double dt, double theta, double mu,
                              int32_t n_controls, const double* u0, const double* z,
                              double newton_tol, double* states);
int tk_forward_burgers_host(int32_t n_steps, int32_t n_u, double dt, double theta, double nu,
                            const double* u0, const double* z, double newton_tol,
                            double* states);
/* Scalar cyclic-reduction coefficients of a symmetric tridiagonal matrix
 * given as [3][n] (sub, diag, sup): out [3][n] = (inv_d, e_up, e_lo) at each
 * node's elimination level.  Host memory. */
int tk_cr_scalar_factor(int32_t n, const double* tri, double* out);
/* Solve with those coefficients (host, for testing the layout). */
int tk_cr_scalar_solve_host(int32_t n, const double* coef, const double* f, double* x);

#ifdef __cplusplus
}
#endif

#endif /* TEMPOKKT_B200_H */
