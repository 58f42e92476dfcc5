// TRI family: partitioned local KKT solves (one CTA per block row, four
// nodes per thread).
//
// Same block-row operation as tri_block (tk_tri.cu; reference kkt.py:298-389
// DiagonalSolver.solve_all, smoothers.py:61-76 jacobi_apply): residual,
// exact solve of the interval's KKT block, update.  Instead of cyclic
// reduction over all n nodes (one barrier per level, half the threads idle
// after the first), the nodes are partitioned into T = 32W contiguous chunks
// of four, one per thread:
//
//   * every thread eliminates its chunk's three interior nodes by two Thomas
//     sweeps in registers: bottom-up (the first interior node in terms of the
//     two chunk interfaces) and top-down (factors T_k = D'_k^{-1} U_k and
//     D'_k^{-1} kept in registers for the back-substitution),
//   * the T interface nodes (the last node of every chunk) form a 2x2-block
//     tridiagonal system, solved by parallel cyclic reduction with a
//     ping-pong shared exchange (one barrier per step),
//   * a forward rhs sweep with the known left interface and a
//     back-substitution recover the interior.
//
// The scalar system Q_z w = r_z rides along through the same steps.  The grid
// is persistent (a few CTAs per SM loop over the block rows), so loads of one
// CTA overlap the solves of the others.  Nodes >= n pad the system to 4T
// nodes with identity blocks.  Node j lives at PI(j) = j + j/16 in the node
// arrays: conflict-free both for the coalesced phases (thread t on node
// t + T s) and the chunk phases (thread t on node 4t + k).
#include "tk_tri.cuh"

namespace tk {

namespace {

constexpr int kChunk = 4;        // nodes per thread
constexpr int kNodeArrays = 7;   // F0 F1 FW KD KS KB SV
constexpr int kXch = 13;         // doubles per thread in one exchange slot

struct S2 { double a, b, c; };   // symmetric [[a b][b c]]

__device__ __forceinline__ S2 inv_s2(double a, double b, double c) {
    const double id = 1.0 / (a * c - b * b);
    return {c * id, -b * id, a * id};
}

}  // namespace

template <int W>
struct PartCta {
    static constexpr int T = 32 * W;          // threads = chunks = interface nodes
    static constexpr int P = kChunk * T;      // padded system size
    static constexpr int PP = P + P / 16 + 1; // padded node-array length
    static constexpr int64_t smem_bytes() {
        return ((int64_t)kNodeArrays * PP + (int64_t)kXch * T) * 8;
    }
    static constexpr int min_blocks() { return W >= 8 ? 1 : 12 / W; }
};

// MODE 0: Jacobi / D^{-1} b (couplings from x through the slab);
// MODE 1 / 2: pass 3 of the forward / backward substitution (coupling from
// the chain vector, no update).
template <int W, int MODE>
__global__ void __launch_bounds__(32 * W, PartCta<W>::min_blocks())
tri_rows_part(TView V, const double* __restrict__ b, const double* __restrict__ x,
              double* __restrict__ y, double omega, const double* __restrict__ chain) {
    using Cf = PartCta<W>;
    constexpr int T = Cf::T, PP = Cf::PP;
    constexpr int NA = kChunk;           // nodes per thread, both layouts
    extern __shared__ __align__(16) double sm[];
    const Lay& L = V.lay;
    const int n = V.n;
    const int tid = threadIdx.x;
    const double kap = V.kappa, k2 = kap * kap;
    const double* Qz = V.Qz;

    double* F0 = sm;
    double* F1 = sm + PP;
    double* FW = sm + 2 * PP;
    double* KD = sm + 3 * PP;   // K diag
    double* KS = sm + 4 * PP;   // K sup  K_{j,j+1}
    double* KB = sm + 5 * PP;   // K sub  K_{j+1,j}
    double* SV = sm + 6 * PP;   // v (coalesced phases)
    double* XB[2] = {KD, sm + kNodeArrays * PP};   // exchange slots (slot 0 over KD..SV)

    const int j0 = kChunk * tid;
    const int64_t bs = V.sl.base;
    for (int i = V.sl.r0 + blockIdx.x; i < V.sl.r1; i += gridDim.x) {
        const bool has_vm = i >= 1, has_uzl = i < L.N;
        const double* Qv = (i == L.N) ? V.Ql : V.Qm;
        const double* Qu = (i == L.N - 1) ? V.Ql : V.Qm;
        const double* K = has_uzl ? V.Ki(i, n) : nullptr;
        const double* C = (has_uzl && has_vm) ? V.Ci(i, n) : nullptr;
        const int64_t ov = L.off_v(i) - bs, ou = L.off_u(i) - bs, oz = L.off_z(i) - bs,
                      om = L.off_mu(i) - bs, ol = L.off_l(i) - bs;
        const double* uprev = nullptr;
        const double* munext = nullptr;
        if (MODE == 0) {
            if (x) { uprev = V.sl.uprev(L, x, i); munext = V.sl.munext(L, x, i); }
        } else if (MODE == 1) {
            if (i >= 1) uprev = chain + (size_t)(i - 1) * n;
        } else {
            if (i < L.N) munext = chain + (size_t)(i + 1) * n;
        }
        const double* xu = MODE == 0 ? x : nullptr;
        const bool hx = MODE == 0 && x != nullptr;

        // ---- phase A (coalesced): residual and K diagonals.  All loads are
        // predicated on warp-uniform flags (no branches), so the compiler can
        // batch them across the NA nodes of a thread.
        double pm[NA];
#pragma unroll
        for (int t = 0; t < NA; ++t) {
            const int j = tid + T * t;
            const bool in = j < n;
            const int jj = in ? j : n - 1;
            const int jm = jj > 0 ? jj - 1 : jj, jp = jj < n - 1 ? jj + 1 : jj;
            const bool lo = in && jj > 0, hi = in && jj < n - 1;
            const bool vm = in && has_vm, uz = in && has_uzl, cc = in && C != nullptr;
            double rv = vm ? b[ov + jj] : 0.0;
            double rm = vm ? b[om + jj] : 0.0;
            double ru = uz ? b[ou + jj] : 0.0;
            double rz = uz ? b[oz + jj] : 0.0;
            double rl = uz ? b[ol + jj] : 0.0;
            const double kd = uz ? K[n + jj] : 0.0;
            const double ks = (uz && hi) ? K[2 * n + jj] : 0.0;
            const double kb = (uz && hi) ? K[jp] : 0.0;
            if (hx) {
                const double ksm = (uz && lo) ? K[2 * n + jm] : 0.0;
                const double kbj = (uz && lo) ? K[jj] : 0.0;
                const double cd = cc ? C[n + jj] : 0.0;
                const double cs = (cc && hi) ? C[2 * n + jj] : 0.0;
                const double cb = (cc && lo) ? C[jj] : 0.0;
                const double csm = (cc && lo) ? C[2 * n + jm] : 0.0;
                const double cbp = (cc && hi) ? C[jp] : 0.0;
                const double xv0 = vm ? x[ov + jj] : 0.0;
                const double xvm = (vm && lo) ? x[ov + jm] : 0.0;
                const double xvp = (vm && hi) ? x[ov + jp] : 0.0;
                const double xm0 = vm ? x[om + jj] : 0.0;
                const double xu0 = uz ? x[ou + jj] : 0.0;
                const double xum = (uz && lo) ? x[ou + jm] : 0.0;
                const double xup = (uz && hi) ? x[ou + jp] : 0.0;
                const double xz0 = uz ? x[oz + jj] : 0.0;
                const double xzm = (uz && lo) ? x[oz + jm] : 0.0;
                const double xzp = (uz && hi) ? x[oz + jp] : 0.0;
                const double xl0 = uz ? x[ol + jj] : 0.0;
                const double xlm = (uz && lo) ? x[ol + jm] : 0.0;
                const double xlp = (uz && hi) ? x[ol + jp] : 0.0;
                const double up = (vm && uprev) ? uprev[jj] : 0.0;
                const double mn = (uz && munext) ? munext[jj] : 0.0;
                // weights (L1-resident)
                const double qvd = Qv[n + jj], qvb = lo ? Qv[jj] : 0.0, qvs = hi ? Qv[2 * n + jj] : 0.0;
                const double qud = Qu[n + jj], qub = lo ? Qu[jj] : 0.0, qus = hi ? Qu[2 * n + jj] : 0.0;
                const double qzd = Qz[n + jj], qzb = lo ? Qz[jj] : 0.0, qzs = hi ? Qz[2 * n + jj] : 0.0;
                if (has_vm) {
                    double av = (qvd * xv0 + qvb * xvm + qvs * xvp) - xm0;
                    av += cd * xl0 + csm * xlm + cbp * xlp;
                    rv -= av;
                    rm += xv0;
                    rm -= up;
                }
                if (has_uzl) {
                    ru -= (qud * xu0 + qub * xum + qus * xup) + (kd * xl0 + ksm * xlm + kb * xlp);
                    ru -= mn;
                    const double qzz = qzd * xz0 + qzb * xzm + qzs * xzp;
                    rz -= qzz + kap * (qzd * xl0 + qzb * xlm + qzs * xlp);
                    double al = (kd * xu0 + kbj * xum + ks * xup) + kap * qzz;
                    al += cd * xv0 + cb * xvm + cs * xvp;
                    rl -= al;
                }
            } else {
                if (vm && uprev) rm -= uprev[jj];
                if (uz && munext) ru -= munext[jj];
            }
            if (!in) { rv = rm = ru = rz = rl = 0.0; }
            const int q = PI(j);
            pm[t] = rv;
            SV[q] = -rm;
            F0[q] = ru;
            F1[q] = rl - kap * rz;
            FW[q] = rz;
            KD[q] = kd;
            KS[q] = ks;
            KB[q] = kb;
        }
        __syncthreads();
        // ---- phase B (coalesced): v, the C v coupling, the mu part without C^T lam
        if (has_vm) {
            double xo[NA], xm[NA];
#pragma unroll
            for (int t = 0; t < NA; ++t) {
                const int j = tid + T * t;
                xo[t] = (xu && j < n) ? xu[ov + j] : 0.0;
                xm[t] = (xu && j < n && !has_uzl) ? xu[om + j] : 0.0;
            }
#pragma unroll
            for (int t = 0; t < NA; ++t) {
                const int j = tid + T * t;
                if (j < n) {
                    const double vj = SV[PI(j)];
                    const double vm = j > 0 ? SV[PI(j - 1)] : 0.0;
                    const double vp = j < n - 1 ? SV[PI(j + 1)] : 0.0;
                    double qv = Qv[n + j] * vj;
                    if (j > 0) qv += Qv[j] * vm;
                    if (j < n - 1) qv += Qv[2 * n + j] * vp;
                    pm[t] = qv - pm[t];
                    if (C) {
                        double cv = C[n + j] * vj;
                        if (j > 0) cv += C[j] * vm;
                        if (j < n - 1) cv += C[2 * n + j] * vp;
                        F1[PI(j)] -= cv;
                    }
                    y[ov + j] = xo[t] + omega * vj;
                    if (!has_uzl) y[om + j] = xm[t] + omega * pm[t];
                }
            }
        }
        if (!has_uzl) {   // last block (v_N, mu_N) is done
            __syncthreads();
            continue;
        }
        __syncthreads();

        // ---- chunk phase.  D_k = [[Qu, K], [K, -k^2 Qz]]_kk,
        // U_k = [[Qu_{k,k+1}, K_{k+1,k}], [K_{k,k+1}, -k^2 Qz_{k,k+1}]]; the
        // scalar system has diagonal Qz_kk and coupling Qz_{k,k+1}.
        auto Dget = [&](int j, double& a, double& bb, double& c) {
            const bool in = j < n;
            a = in ? Qu[n + j] : 1.0;
            bb = KD[PI(j)];
            c = in ? -k2 * Qz[n + j] : -1.0;
        };
        auto Uget = [&](int j, double& u0, double& u1, double& u2, double& u3) {
            const bool cpl = j >= 0 && j < n - 1;
            u0 = cpl ? Qu[2 * n + j] : 0.0;
            u1 = cpl ? KB[PI(j)] : 0.0;
            u2 = cpl ? KS[PI(j)] : 0.0;
            u3 = cpl ? -k2 * Qz[2 * n + j] : 0.0;
        };
        auto dzs = [&](int j) -> double { return j < n ? Qz[n + j] : 1.0; };
        auto ezs = [&](int j) -> double { return (j >= 0 && j < n - 1) ? Qz[2 * n + j] : 0.0; };

        double fa[NA], fb[NA], fw[NA];
#pragma unroll
        for (int k = 0; k < NA; ++k) {
            const int q = PI(j0 + k);
            fa[k] = F0[q];
            fb[k] = F1[q];
            fw[k] = FW[q];
        }
        // couplings needed after the exchange slot 0 (over KD..SV) is reused
        double ul0, ul1, ul2, ul3, ur0, ur1, ur2, ur3;
        Uget(j0 - 1, ul0, ul1, ul2, ul3);            // left interface -> node 0
        Uget(j0 + NA - 1, ur0, ur1, ur2, ur3);       // own interface -> next chunk
        const double sel = ezs(j0 - 1), ser = ezs(j0 + NA - 1);

        // step A (bottom-up over the interior): y_0 = iDh (h + H x_R - U_{-1}^T x_L)
        double ha, hb, H00, H01, H10, H11;
        S2 iDh;
        double s_idh, s_hh, s_Hh;
        {
            double da, db, dc;
            Dget(j0 + NA - 2, da, db, dc);
            ha = fa[NA - 2];
            hb = fb[NA - 2];
            double u0, u1, u2, u3;
            Uget(j0 + NA - 2, u0, u1, u2, u3);
            H00 = -u0; H01 = -u1; H10 = -u2; H11 = -u3;
            double sd = dzs(j0 + NA - 2);
            s_hh = fw[NA - 2];
            s_Hh = -ezs(j0 + NA - 2);
#pragma unroll
            for (int k = NA - 2; k >= 1; --k) {
                const S2 iv = inv_s2(da, db, dc);
                Uget(j0 + k - 1, u0, u1, u2, u3);
                const double s00 = iv.a * u0 + iv.b * u1, s01 = iv.a * u2 + iv.b * u3;
                const double s10 = iv.b * u0 + iv.c * u1, s11 = iv.b * u2 + iv.c * u3;
                double a, bb, c;
                Dget(j0 + k - 1, a, bb, c);
                da = a - (u0 * s00 + u1 * s10);
                db = bb - (u0 * s01 + u1 * s11);
                dc = c - (u2 * s01 + u3 * s11);
                const double nha = fa[k - 1] - (s00 * ha + s10 * hb);
                const double nhb = fb[k - 1] - (s01 * ha + s11 * hb);
                ha = nha; hb = nhb;
                const double n00 = -(s00 * H00 + s10 * H10), n01 = -(s00 * H01 + s10 * H11);
                const double n10 = -(s01 * H00 + s11 * H10), n11 = -(s01 * H01 + s11 * H11);
                H00 = n00; H01 = n01; H10 = n10; H11 = n11;
                // scalar
                const double e = ezs(j0 + k - 1);
                const double sb = e / sd;
                sd = dzs(j0 + k - 1) - e * sb;
                s_hh = fw[k - 1] - sb * s_hh;
                s_Hh = -sb * s_Hh;
            }
            iDh = inv_s2(da, db, dc);
            s_idh = 1.0 / sd;
        }
        // step B (top-down): T_k, D'_k^{-1} in registers
        double Tt[NA - 1][4], Ti[NA - 1][3], st[NA - 1], sid[NA - 1];
        double pa, pb, pc, ga, gb, F00, F01, F10, F11, s_dp, s_g, s_F;
        {
            Dget(j0, pa, pb, pc);
            ga = fa[0];
            gb = fb[0];
            F00 = -ul0; F01 = -ul2; F10 = -ul1; F11 = -ul3;
            s_dp = dzs(j0);
            s_g = fw[0];
            s_F = -sel;
#pragma unroll
            for (int k = 1; k < NA; ++k) {
                const S2 iv = inv_s2(pa, pb, pc);
                double u0, u1, u2, u3;
                Uget(j0 + k - 1, u0, u1, u2, u3);
                const double t00 = iv.a * u0 + iv.b * u2, t01 = iv.a * u1 + iv.b * u3;
                const double t10 = iv.b * u0 + iv.c * u2, t11 = iv.b * u1 + iv.c * u3;
                Tt[k - 1][0] = t00; Tt[k - 1][1] = t01; Tt[k - 1][2] = t10; Tt[k - 1][3] = t11;
                Ti[k - 1][0] = iv.a; Ti[k - 1][1] = iv.b; Ti[k - 1][2] = iv.c;
                double a, bb, c;
                Dget(j0 + k, a, bb, c);
                pa = a - (u0 * t00 + u2 * t10);
                pb = bb - (u0 * t01 + u2 * t11);
                pc = c - (u1 * t01 + u3 * t11);
                const double nga = fa[k] - (t00 * ga + t10 * gb);
                const double ngb = fb[k] - (t01 * ga + t11 * gb);
                ga = nga; gb = ngb;
                const double n00 = -(t00 * F00 + t10 * F10), n01 = -(t00 * F01 + t10 * F11);
                const double n10 = -(t01 * F00 + t11 * F10), n11 = -(t01 * F01 + t11 * F11);
                F00 = n00; F01 = n01; F10 = n10; F11 = n11;
                // scalar
                const double e = ezs(j0 + k - 1);
                const double tt = e / s_dp;
                st[k - 1] = tt;
                sid[k - 1] = 1.0 / s_dp;
                s_dp = dzs(j0 + k) - e * tt;
                s_g = fw[k] - tt * s_g;
                s_F = -tt * s_F;
            }
        }
        __syncthreads();   // KD..SV are dead: exchange slot 0 may overwrite them
        // exchange 1: this chunk's bottom-up results for the previous chunk
        {
            double* E = XB[0];
            E[0 * T + tid] = iDh.a; E[1 * T + tid] = iDh.b; E[2 * T + tid] = iDh.c;
            E[3 * T + tid] = ha; E[4 * T + tid] = hb;
            E[5 * T + tid] = H00; E[6 * T + tid] = H01; E[7 * T + tid] = H10; E[8 * T + tid] = H11;
            E[9 * T + tid] = s_idh; E[10 * T + tid] = s_hh; E[11 * T + tid] = s_Hh;
        }
        __syncthreads();
        // step C: interface rows  A X_{l-1} + B X_l + C X_{l+1} = R  (block and scalar)
        double B00, B01, B10, B11, C00, C01, C10, C11, A00, A01, A10, A11, R0, R1;
        double sA, sB, sC, sR;
        {
            const double* E = XB[0];
            const int nx = tid + 1 < T ? tid + 1 : tid;   // last chunk: coupling is zero
            const double na = E[0 * T + nx], nb = E[1 * T + nx], nc = E[2 * T + nx];
            const double nha = E[3 * T + nx], nhb = E[4 * T + nx];
            const double nH00 = E[5 * T + nx], nH01 = E[6 * T + nx];
            const double nH10 = E[7 * T + nx], nH11 = E[8 * T + nx];
            const double nsi = E[9 * T + nx], nsh = E[10 * T + nx], nsH = E[11 * T + nx];
            const double v00 = ur0 * na + ur1 * nb, v01 = ur0 * nb + ur1 * nc;
            const double v10 = ur2 * na + ur3 * nb, v11 = ur2 * nb + ur3 * nc;
            B00 = pa - (v00 * ur0 + v01 * ur1); B01 = pb - (v00 * ur2 + v01 * ur3);
            B10 = pb - (v10 * ur0 + v11 * ur1); B11 = pc - (v10 * ur2 + v11 * ur3);
            C00 = v00 * nH00 + v01 * nH10; C01 = v00 * nH01 + v01 * nH11;
            C10 = v10 * nH00 + v11 * nH10; C11 = v10 * nH01 + v11 * nH11;
            A00 = -F00; A01 = -F01; A10 = -F10; A11 = -F11;
            R0 = ga - (v00 * nha + v01 * nhb);
            R1 = gb - (v10 * nha + v11 * nhb);
            const double rho = ser * nsi;
            sA = -s_F;
            sB = s_dp - ser * rho;
            sC = rho * nsH;
            sR = s_g - rho * nsh;
        }
        // parallel cyclic reduction over the T interface rows (ping-pong slots)
        int slot = 1;
#pragma unroll
        for (int s = 1; s < T; s <<= 1) {
            const double id = 1.0 / (B00 * B11 - B01 * B10);
            const double i00 = B11 * id, i01 = -B01 * id, i10 = -B10 * id, i11 = B00 * id;
            const double isb = 1.0 / sB;
            double* E = XB[slot];
            E[0 * T + tid] = i00 * A00 + i01 * A10; E[1 * T + tid] = i00 * A01 + i01 * A11;
            E[2 * T + tid] = i10 * A00 + i11 * A10; E[3 * T + tid] = i10 * A01 + i11 * A11;
            E[4 * T + tid] = i00 * C00 + i01 * C10; E[5 * T + tid] = i00 * C01 + i01 * C11;
            E[6 * T + tid] = i10 * C00 + i11 * C10; E[7 * T + tid] = i10 * C01 + i11 * C11;
            E[8 * T + tid] = i00 * R0 + i01 * R1;   E[9 * T + tid] = i10 * R0 + i11 * R1;
            E[10 * T + tid] = isb * sA; E[11 * T + tid] = isb * sC; E[12 * T + tid] = isb * sR;
            __syncthreads();
            double mc00 = 0, mc01 = 0, mc10 = 0, mc11 = 0, ma00 = 0, ma01 = 0, ma10 = 0, ma11 = 0;
            double mr0 = 0, mr1 = 0, msa = 0, msc = 0, msr = 0;
            double pa00 = 0, pa01 = 0, pa10 = 0, pa11 = 0, pc00 = 0, pc01 = 0, pc10 = 0, pc11 = 0;
            double pr0 = 0, pr1 = 0, psa = 0, psc = 0, psr = 0;
            if (tid >= s) {
                const int m = tid - s;
                ma00 = E[0 * T + m]; ma01 = E[1 * T + m]; ma10 = E[2 * T + m]; ma11 = E[3 * T + m];
                mc00 = E[4 * T + m]; mc01 = E[5 * T + m]; mc10 = E[6 * T + m]; mc11 = E[7 * T + m];
                mr0 = E[8 * T + m]; mr1 = E[9 * T + m];
                msa = E[10 * T + m]; msc = E[11 * T + m]; msr = E[12 * T + m];
            }
            if (tid + s < T) {
                const int m = tid + s;
                pa00 = E[0 * T + m]; pa01 = E[1 * T + m]; pa10 = E[2 * T + m]; pa11 = E[3 * T + m];
                pc00 = E[4 * T + m]; pc01 = E[5 * T + m]; pc10 = E[6 * T + m]; pc11 = E[7 * T + m];
                pr0 = E[8 * T + m]; pr1 = E[9 * T + m];
                psa = E[10 * T + m]; psc = E[11 * T + m]; psr = E[12 * T + m];
            }
            // B -= A (iB C)_{l-s} + C (iB A)_{l+s};  A <- -A (iB A)_{l-s};  C <- -C (iB C)_{l+s}
            B00 -= (A00 * mc00 + A01 * mc10) + (C00 * pa00 + C01 * pa10);
            B01 -= (A00 * mc01 + A01 * mc11) + (C00 * pa01 + C01 * pa11);
            B10 -= (A10 * mc00 + A11 * mc10) + (C10 * pa00 + C11 * pa10);
            B11 -= (A10 * mc01 + A11 * mc11) + (C10 * pa01 + C11 * pa11);
            R0 -= (A00 * mr0 + A01 * mr1) + (C00 * pr0 + C01 * pr1);
            R1 -= (A10 * mr0 + A11 * mr1) + (C10 * pr0 + C11 * pr1);
            const double nA00 = -(A00 * ma00 + A01 * ma10), nA01 = -(A00 * ma01 + A01 * ma11);
            const double nA10 = -(A10 * ma00 + A11 * ma10), nA11 = -(A10 * ma01 + A11 * ma11);
            const double nC00 = -(C00 * pc00 + C01 * pc10), nC01 = -(C00 * pc01 + C01 * pc11);
            const double nC10 = -(C10 * pc00 + C11 * pc10), nC11 = -(C10 * pc01 + C11 * pc11);
            A00 = nA00; A01 = nA01; A10 = nA10; A11 = nA11;
            C00 = nC00; C01 = nC01; C10 = nC10; C11 = nC11;
            sB -= sA * msc + sC * psa;
            sR -= sA * msr + sC * psr;
            sA = -sA * msa;
            sC = -sC * psc;
            slot ^= 1;
        }
        double X0, X1, sX;
        {
            const double id = 1.0 / (B00 * B11 - B01 * B10);
            X0 = (B11 * R0 - B01 * R1) * id;
            X1 = (B00 * R1 - B10 * R0) * id;
            sX = sR / sB;
        }
        // exchange 2: interface values for the next chunk
        {
            double* E = XB[slot];
            E[tid] = X0; E[T + tid] = X1; E[2 * T + tid] = sX;
        }
        __syncthreads();
        double xl0 = 0.0, xl1 = 0.0, sxl = 0.0;
        if (tid > 0) {
            const double* E = XB[slot];
            xl0 = E[tid - 1]; xl1 = E[T + tid - 1]; sxl = E[2 * T + tid - 1];
        }
        // steps D/E: rhs sweep with the left interface, back-substitution
        {
            double g0[NA - 1], g1[NA - 1], gs[NA - 1];
#pragma unroll
            for (int k = 0; k < NA - 1; ++k) {   // rhs again from the node arrays
                const int q = PI(j0 + k);
                g0[k] = F0[q];
                g1[k] = F1[q];
                gs[k] = FW[q];
            }
            g0[0] -= ul0 * xl0 + ul2 * xl1;
            g1[0] -= ul1 * xl0 + ul3 * xl1;
            gs[0] -= sel * sxl;
#pragma unroll
            for (int k = 1; k < NA - 1; ++k) {
                const double* t = Tt[k - 1];
                g0[k] -= t[0] * g0[k - 1] + t[2] * g1[k - 1];
                g1[k] -= t[1] * g0[k - 1] + t[3] * g1[k - 1];
                gs[k] -= st[k - 1] * gs[k - 1];
            }
            double ya = X0, yb = X1, ys = sX;
            {
                const int q = PI(j0 + NA - 1);
                F0[q] = X0; F1[q] = X1; FW[q] = sX;
            }
#pragma unroll
            for (int k = NA - 2; k >= 0; --k) {
                const double* t = Tt[k];
                const double* iv = Ti[k];
                const double na = iv[0] * g0[k] + iv[1] * g1[k] - (t[0] * ya + t[1] * yb);
                const double nb = iv[1] * g0[k] + iv[2] * g1[k] - (t[2] * ya + t[3] * yb);
                ys = sid[k] * gs[k] - st[k] * ys;
                ya = na; yb = nb;
                const int q = PI(j0 + k);
                F0[q] = na; F1[q] = nb; FW[q] = ys;
            }
        }
        __syncthreads();
        // ---- output (coalesced)
        {
            double xo[NA][5];
#pragma unroll
            for (int t = 0; t < NA; ++t) {
                const int j = tid + T * t;
                const bool in = xu && j < n;
                xo[t][0] = in ? xu[ou + j] : 0.0;
                xo[t][1] = in ? xu[oz + j] : 0.0;
                xo[t][2] = in ? xu[ol + j] : 0.0;
                xo[t][3] = (in && has_vm) ? xu[om + j] : 0.0;
            }
#pragma unroll
            for (int t = 0; t < NA; ++t) {
                const int j = tid + T * t;
                if (j < n) {
                    const int q = PI(j);
                    const double du = F0[q], dl = F1[q];
                    const double dzv = FW[q] - kap * dl;
                    y[ou + j] = xo[t][0] + omega * du;
                    y[oz + j] = xo[t][1] + omega * dzv;
                    y[ol + j] = xo[t][2] + omega * dl;
                    if (has_vm) {
                        double dm = pm[t];
                        if (C) {
                            dm += C[n + j] * dl;
                            if (j > 0) dm += C[2 * n + j - 1] * F1[PI(j - 1)];
                            if (j < n - 1) dm += C[j + 1] * F1[PI(j + 1)];
                        }
                        y[om + j] = xo[t][3] + omega * dm;
                    }
                }
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// host dispatch
// ---------------------------------------------------------------------------
static int part_warps(int n) {
    if (n <= 4 || n > 2048) return 0;
    int w = 1;
    while (kChunk * 32 * w < n) w <<= 1;
    return w;
}

int part_nodes_per_lane(int n) { return part_warps(n) ? kChunk : 0; }

template <int W, int MODE>
static int part_launch_t(const tk_level* Lv, const double* b, const double* x, double* y,
                         double omega, const double* chain, cudaStream_t s) {
    using Cf = PartCta<W>;
    static int per_sm = 0;
    static int nsm = 0;
    const int64_t smem = Cf::smem_bytes();
    if (!per_sm) {
        cudaFuncSetAttribute(tri_rows_part<W, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        cudaFuncSetAttribute(tri_rows_part<W, MODE>, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared);
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        int per = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, tri_rows_part<W, MODE>, 32 * W,
                                                      (size_t)smem);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_status(e, "tri_rows_part: attributes");
        if (per < 1) {
            set_error("tri_rows_part<%d>: does not fit on an SM (%lld B smem)", W, (long long)smem);
            return TK_ERR_CUDA;
        }
        per_sm = per;
    }
    TView V(Lv);
    const int rows = V.sl.r1 - V.sl.r0;
    int grid = rows;
    const int cap = nsm * per_sm;
    if (grid > cap) grid = cap;
    tri_rows_part<W, MODE><<<grid, 32 * W, smem, s>>>(V, b, x, y, omega, chain);
    return check_launch("tri_rows_part");
}

// mode 0: rows (jacobi / D^{-1} b), 1/2: substitution pass 3 forward/backward
int part_launch(const tk_level* Lv, int mode, const double* b, const double* x, double* y,
                double omega, const double* chain, cudaStream_t s) {
#define TK_PART_CASE(WW)                                                              \
    case WW:                                                                          \
        if (mode == 0) return part_launch_t<WW, 0>(Lv, b, x, y, omega, chain, s);     \
        if (mode == 1) return part_launch_t<WW, 1>(Lv, b, x, y, omega, chain, s);     \
        return part_launch_t<WW, 2>(Lv, b, x, y, omega, chain, s);
    switch (part_warps(Lv->n_u)) {
        TK_PART_CASE(1)
        TK_PART_CASE(2)
        TK_PART_CASE(4)
        TK_PART_CASE(8)
        TK_PART_CASE(16)
        default: set_error("tri_rows_part: unsupported n_u=%d", Lv->n_u); return TK_ERR_UNSUPPORTED;
    }
#undef TK_PART_CASE
}

}  // namespace tk
