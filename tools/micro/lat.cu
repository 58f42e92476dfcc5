// fp64 / shared-memory latency microbenchmarks (one warp): nvcc -arch=sm_100a -O3 lat.cu -o lat
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double a, double b) {
    __shared__ double2 sm[64];
    double x = out[threadIdx.x], y = out[32 + threadIdx.x];
    long long c0, c1;
    // 1: dependent DFMA chain
    c0 = clock64();
#pragma unroll
    for (int i = 0; i < 256; ++i) x = fma(x, a, b);
    c1 = clock64();
    if (threadIdx.x == 0) cyc[0] = c1 - c0;
    // 2: two independent DFMA chains
    c0 = clock64();
#pragma unroll
    for (int i = 0; i < 256; ++i) { x = fma(x, a, b); y = fma(y, a, b); }
    c1 = clock64();
    if (threadIdx.x == 0) cyc[1] = c1 - c0;
    // 3: dependent DADD
    c0 = clock64();
#pragma unroll
    for (int i = 0; i < 256; ++i) x = x + a;
    c1 = clock64();
    if (threadIdx.x == 0) cyc[2] = c1 - c0;
    // 4: STS -> syncwarp -> LDS round trip, dependent
    c0 = clock64();
#pragma unroll
    for (int i = 0; i < 64; ++i) {
        sm[threadIdx.x] = make_double2(x, y);
        __syncwarp();
        const double2 v = sm[(threadIdx.x + 1) & 31];
        __syncwarp();
        x = v.x; y = v.y;
    }
    c1 = clock64();
    if (threadIdx.x == 0) cyc[3] = c1 - c0;
    // 5: 8 independent DFMA chains
    double z[8];
    for (int j = 0; j < 8; ++j) z[j] = x + j;
    c0 = clock64();
#pragma unroll
    for (int i = 0; i < 64; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) z[j] = fma(z[j], a, b);
    c1 = clock64();
    if (threadIdx.x == 0) cyc[4] = c1 - c0;
    for (int j = 0; j < 8; ++j) x += z[j];
    // 6: shuffle round trip (double = 2 shuffles), dependent
    c0 = clock64();
#pragma unroll
    for (int i = 0; i < 64; ++i) x = __shfl_down_sync(0xffffffffu, x, 1) + a;
    c1 = clock64();
    if (threadIdx.x == 0) cyc[5] = c1 - c0;
    // 7: dependent LDS chain (pointer chase through shared)
    __shared__ int idx[32];
    idx[threadIdx.x] = (threadIdx.x + 1) & 31;
    __syncwarp();
    int p = threadIdx.x;
    c0 = clock64();
#pragma unroll
    for (int i = 0; i < 64; ++i) p = idx[p];
    c1 = clock64();
    if (threadIdx.x == 0) cyc[6] = c1 - c0;
    out[threadIdx.x] = x + y + p;
}
int main() {
    double* d; long long* c;
    cudaMalloc(&d, 64 * 8); cudaMemset(d, 0, 64 * 8);
    cudaMalloc(&c, 8 * 8);
    for (int r = 0; r < 2; ++r) k<<<1, 32>>>(d, c, 1.0000001, 1e-9);
    long long h[8];
    cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
    printf("dep DFMA %.1f cyc/op | 2 chains %.1f cyc/pair | dep DADD %.1f | STS-sync-LDS-sync %.1f | 8 chains %.1f cyc/round | shfl+dadd %.1f | dep LDS %.1f\n",
           h[0] / 256.0, h[1] / 256.0, h[2] / 256.0, h[3] / 64.0, h[4] / 64.0, h[5] / 64.0, h[6] / 64.0);
    return 0;
}
