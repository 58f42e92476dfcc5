// TRI family: partitioned local KKT solves -- host dispatch (the kernels live in
// tk_tri_part.cuh; each row width is instantiated in tk_tri_part_w*.cu).
#define TK_PART_MAIN_TU
#include "tk_tri_part.cuh"

namespace tk {

#define TK_PART_EXTERN(WW, CC)                                                                       \
    extern template int part_dispatch_x<WW, CC>(const tk_level*, int, bool, const double*,          \
                                                const double*, double*, double, const double*,      \
                                                cudaStream_t, double*, const double*, int);
#define TK_PART_EXTERN_R(WW, CC)                                                                     \
    extern template int part_dispatch_r<WW, CC>(const tk_level*, bool, const double*, const double*, \
                                                double*, double, const double*, cudaStream_t);
TK_PART_EXTERN(1, 1) TK_PART_EXTERN(2, 1) TK_PART_EXTERN(4, 1) TK_PART_EXTERN(8, 1) TK_PART_EXTERN(16, 1)
TK_PART_EXTERN_R(1, 1) TK_PART_EXTERN_R(2, 1) TK_PART_EXTERN_R(4, 1) TK_PART_EXTERN_R(8, 1)
TK_PART_EXTERN_R(8, 2)

// mode 0: rows (jacobi / D^{-1} b), 1/2: substitution pass 3 forward/backward;
// rc: the zero-start sweep also writes its restricted residual (opt bit 0:
// only the u and mu segments of y are stored); ec (mode 0, omega == 1): the
// couplings are those of x + P ec (the V-cycle's prolongation fused into the
// post-smoothing sweep)
int part_launch(const tk_level* Lv, int mode, const double* b, const double* x, double* y,
                double omega, const double* chain, cudaStream_t s, double* rc, const double* ec,
                int opt) {
#define TK_PART_X(WW, CC)                                                                           \
    if (mode != 0 && w == WW && cl == CC) {                                                         \
        const int r_ = part_dispatch_x<WW, CC>(Lv, mode, full, b, x, y, omega, chain, s, rc, ec, opt); \
        if (r_ != -1) return r_;                                                                    \
    }
#define TK_PART_R(WW, CC)                                                                           \
    if (mode == 0 && w == WW && cl == CC)                                                           \
        return part_dispatch_r<WW, CC>(Lv, full, b, x, y, omega, chain, s);
    // Jacobi with omega == 1 or from zero needs x only through the two
    // continuity couplings: x + D^{-1}(b - A x) = D^{-1}(b + (L + U) x), the
    // local solve of b with u_{i-1} / mu_{i+1} moved to the right-hand side
    // (MODE 3: no D x products, no second read of x; 164 / 128 instead of 232
    // registers).  TK_JACOBI_RESIDUAL_FORM=1 keeps the residual form.
    static const bool resid_form = [] {
        const char* e = getenv("TK_JACOBI_RESIDUAL_FORM");
        return e && e[0] == '1';
    }();
    if (mode == 0 && (x == nullptr || (omega == 1.0 && !resid_form))) mode = 3;
    // FULL: every chunk is complete and every segment 16-byte aligned
    const int w = part_warps(Lv->n_u, mode), cl = part_cluster(Lv->n_u, mode);
    auto al = [](const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    // a whole level with even N, or a time slab cut at even rows
    const int r1 = Lv->row1 > 0 ? Lv->row1 : Lv->n_steps + 1;
    const bool slab_even = (Lv->n_steps & 1) == 0 && (Lv->row0 & 1) == 0 &&
                           (r1 == Lv->n_steps + 1 || (r1 & 1) == 0) && r1 - Lv->row0 >= 2;
    const bool whole = Lv->row0 == 0 && r1 == Lv->n_steps + 1;
    if (rc && !ec && (mode != 3 || omega != 1.0 || !slab_even || (x && (opt & 1)))) {
        set_error("tri_rows_part: the fused restriction needs a sweep with omega = 1 on a level "
                  "(or slab cut at even rows) with even N (partial output only from zero)");
        return TK_ERR_UNSUPPORTED;
    }
    const bool full = w > 0 && Lv->n_u == kChunk * 32 * w * cl && Lv->n_u % 2 == 0 && Lv->n_z % 2 == 0 &&
                      al(b) && al(x) && al(y) && al(chain) && al(rc) && al(ec) && al(Lv->K) &&
                      al(Lv->C) && al(Lv->Qm) && al(Lv->Ql) && al(Lv->Qz) && al(Lv->halo_u) &&
                      al(Lv->halo_mu);
    if (ec && (mode != 3 || !x || !slab_even || w == 0 || cl != 1 || (!whole && !rc))) {
        set_error("tri_rows_part: the fused prolongation needs omega = 1, x and a level (or slab "
                  "cut at even rows, with its coarse halos) with even N");
        return TK_ERR_UNSUPPORTED;
    }
    TK_PART_X(1, 1)
    TK_PART_X(2, 1)
    TK_PART_X(4, 1)
    TK_PART_X(8, 1)
    TK_PART_X(16, 1)
    TK_PART_R(1, 1)
    TK_PART_R(2, 1)
    TK_PART_R(4, 1)
    TK_PART_R(8, 1)
    TK_PART_R(8, 2)
#undef TK_PART_X
#undef TK_PART_R
    set_error("tri_rows_part: unsupported n_u=%d", Lv->n_u);
    return TK_ERR_UNSUPPORTED;
}

// whether tk_jacobi_prolong's fused rows cover the level (any 4 < n_u <= 2048: rows that
// are not full multiples of the chunk count take the guarded loads)
bool part_full_rows(const tk_level* Lv) {
    return part_warps(Lv->n_u, 3) > 0 && part_cluster(Lv->n_u, 3) == 1;
}

}  // namespace tk
