// Time-level transfers on the reference layout (multigrid.py:263-300):
// states/multipliers (u, v, lam, mu) use injection down / linear interpolation
// up; piecewise-constant controls use 2-interval averages down / copies up.
// One thread per (time index, slot); a slot enumerates the 4nu+nz variables
// of one time index: [u | v | z | mu | lam].
#include "tk_common.cuh"

namespace tk {

__device__ __forceinline__ int64_t slot_off(const Lay& L, int t, int slot, bool& is_z) {
    const int nu = L.nu, nz = L.nz;
    is_z = false;
    if (slot < nu) return L.t_u(t) + slot;
    slot -= nu;
    if (slot < nu) return L.t_v(t) + slot;
    slot -= nu;
    if (slot < nz) { is_z = true; return L.t_z(t) + slot; }
    slot -= nz;
    if (slot < nu) return L.t_mu(t) + slot;
    slot -= nu;
    return L.t_l(t) + slot;
}

__global__ void restrict_kernel(Lay Lf, Lay Lc, const double* __restrict__ xf,
                                double* __restrict__ xc) {
    const int64_t m = Lc.m;
    const int64_t total = (int64_t)Lc.N * m;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int t = (int)(k / m) + 1;
        const int slot = (int)(k % m);
        bool is_z;
        const int64_t oc = slot_off(Lc, t, slot, is_z);
        if (is_z) {
            const int64_t a = slot_off(Lf, 2 * t - 1, slot, is_z);
            const int64_t b = slot_off(Lf, 2 * t, slot, is_z);
            xc[oc] = 0.5 * (xf[a] + xf[b]);
        } else {
            xc[oc] = xf[slot_off(Lf, 2 * t, slot, is_z)];
        }
    }
}

__global__ void prolong_add_kernel(Lay Lf, Lay Lc, const double* __restrict__ xc,
                                   double* __restrict__ xf) {
    const int64_t m = Lf.m;
    const int64_t total = (int64_t)Lf.N * m;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int t = (int)(k / m) + 1;
        const int slot = (int)(k % m);
        bool is_z;
        const int64_t of = slot_off(Lf, t, slot, is_z);
        double val;
        if (is_z) {
            val = xc[slot_off(Lc, (t + 1) / 2, slot, is_z)];
        } else if ((t & 1) == 0) {
            val = xc[slot_off(Lc, t / 2, slot, is_z)];
        } else if (t == 1) {
            val = xc[slot_off(Lc, 1, slot, is_z)];
        } else {
            const int j = (t - 1) / 2;
            val = 0.5 * (xc[slot_off(Lc, j, slot, is_z)] + xc[slot_off(Lc, j + 1, slot, is_z)]);
        }
        xf[of] = xf[of] + val;
    }
}

int transfer_launch(int restrict_op, int n_fine, int nu, int nz, const double* in, double* out,
                    cudaStream_t s) {
    Lay Lf(n_fine, nu, nz), Lc(n_fine / 2, nu, nz);
    const int th = 256;
    if (restrict_op) {
        restrict_kernel<<<grid_for(Lc.dim(), th, 148 * 32), th, 0, s>>>(Lf, Lc, in, out);
    } else {
        prolong_add_kernel<<<grid_for(Lf.dim(), th, 148 * 32), th, 0, s>>>(Lf, Lc, in, out);
    }
    return check_launch("transfer");
}

}  // namespace tk
