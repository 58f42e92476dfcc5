// Stage linearisation on the device (timedisc.py:133-149 via kkt.py:100-124):
//   K_i = -M + dt*theta*F_u(u_i, z_i)
//   C_i =  M + dt*(1-theta)*F_u(v_{i-1}, z_i),  v_{-1} = u0
//   B_i = dt*theta*F_z + dt*(1-theta)*F_z
// Products and sums use explicit round-to-nearest intrinsics (no FMA
// contraction) in numpy's evaluation order, so the stage data match the
// reference's bit for bit.
#include "tk_common.cuh"

namespace tk {

__device__ __forceinline__ double M_(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double A_(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double S_(double a, double b) { return __dsub_rn(a, b); }

// F_u of van der Pol (problems.py:56-60)
__device__ __forceinline__ void vdp_fu(double mu, const double* u, double f[4]) {
    f[0] = 0.0;
    f[1] = 1.0;
    f[2] = S_(M_(M_(M_(-2.0, mu), u[0]), u[1]), 1.0);
    f[3] = M_(mu, S_(1.0, M_(u[0], u[0])));
}

__global__ void stage_vdp_kernel(int N, double dt, double theta, double mu, int nc,
                                 const double* __restrict__ u0, const double* __restrict__ u,
                                 const double* __restrict__ v, const double* __restrict__ z,
                                 double* __restrict__ K, double* __restrict__ C,
                                 double* __restrict__ B) {
    const double ct = M_(dt, theta);
    const double cc = M_(dt, S_(1.0, theta));
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
        const double* ui = u + 2 * i;
        const double* vp = (i == 0) ? u0 : v + 2 * (i - 1);
        double fk[4], fc[4];
        vdp_fu(mu, ui, fk);
        vdp_fu(mu, vp, fc);
        const double eye[4] = {1.0, 0.0, 0.0, 1.0};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            K[4 * i + e] = A_(-eye[e], M_(ct, fk[e]));
            C[4 * i + e] = A_(eye[e], M_(cc, fc[e]));
        }
        if (nc == 2) {
#pragma unroll
            for (int e = 0; e < 4; ++e) B[4 * i + e] = A_(M_(ct, eye[e]), M_(cc, eye[e]));
        } else {
            B[2 * i + 0] = A_(M_(ct, 0.0), M_(cc, 0.0));
            B[2 * i + 1] = A_(M_(ct, 1.0), M_(cc, 1.0));
        }
    }
}

// Burgers F_u = -nu*A_stiff - J_conv(u) (problems.py:127-138, 166-167),
// P1 elements on n interior nodes, h = 1/(n+1).  Writes diagonals of
// out = sgn*M + c*F_u(w) as [3][n].
__device__ __forceinline__ void burgers_row(int n, double h, double nu, const double* w, int j,
                                            double sgn, double c, double* out) {
    const double hs = h / 6.0, hd = (4.0 * h) / 6.0;
    const double st_o = M_(-nu, -1.0 / h), st_d = M_(-nu, 2.0 / h);
    const double uj = w[j];
    const double up = (j < n - 1) ? w[j + 1] : 0.0;
    const double um = (j > 0) ? w[j - 1] : 0.0;
    const double d = S_(up, um) / 6.0;
    const double fd = S_(st_d, d);
    out[n + j] = A_(sgn * hd, M_(c, fd));
    if (j > 0) {
        const double lo = S_(-uj, M_(2.0, um)) / 6.0;
        out[j] = A_(sgn * hs, M_(c, S_(st_o, lo)));
    } else {
        out[j] = 0.0;
    }
    if (j < n - 1) {
        const double hi = A_(M_(2.0, up), uj) / 6.0;
        out[2 * n + j] = A_(sgn * hs, M_(c, S_(st_o, hi)));
    } else {
        out[2 * n + j] = 0.0;
    }
}

__global__ void stage_burgers_kernel(int N, int n, double dt, double theta, double nu,
                                     const double* __restrict__ u0, const double* __restrict__ u,
                                     const double* __restrict__ v, double* __restrict__ K,
                                     double* __restrict__ C) {
    const double h = 1.0 / (double)(n + 1);
    const double ct = M_(dt, theta);
    const double cc = M_(dt, S_(1.0, theta));
    for (int i = blockIdx.x; i < N; i += gridDim.x) {
        const double* ui = u + (size_t)i * n;
        const double* vp = (i == 0) ? u0 : v + (size_t)(i - 1) * n;
        for (int j = threadIdx.x; j < n; j += blockDim.x) {
            burgers_row(n, h, nu, ui, j, -1.0, ct, K + (size_t)i * 3 * n);
            burgers_row(n, h, nu, vp, j, 1.0, cc, C + (size_t)i * 3 * n);
        }
    }
}

int stage_vdp_launch(int N, double dt, double theta, double mu, int nc, const double* u0,
                     const double* u, const double* v, const double* z, double* K, double* C,
                     double* B, cudaStream_t s) {
    stage_vdp_kernel<<<grid_for(N, 128, 1 << 20), 128, 0, s>>>(N, dt, theta, mu, nc, u0, u, v, z,
                                                               K, C, B);
    return check_launch("stage_vdp");
}

int stage_burgers_launch(int N, int n, double dt, double theta, double nu, const double* u0,
                         const double* u, const double* v, double* K, double* C,
                         cudaStream_t s) {
    const int th = n >= 256 ? 256 : 128;
    stage_burgers_kernel<<<N < (1 << 30) ? N : (1 << 30), th, 0, s>>>(N, n, dt, theta, nu, u0, u,
                                                                       v, K, C);
    return check_launch("stage_burgers");
}

}  // namespace tk
