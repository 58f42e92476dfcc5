// fp64 issue throughput per warp / per SM partition (B200): ./dpthr
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k(double* out, int iters, double a, double b) {
    double z[CH];
#pragma unroll
    for (int j = 0; j < CH; ++j) z[j] = out[threadIdx.x] + j;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int j = 0; j < CH; ++j) z[j] = fma(z[j], a, b);
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < CH; ++j) s += z[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int CH>
void run(int warps, double* d) {
    const int iters = 20000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<CH><<<1, 32 * warps>>>(d, 100, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    k<CH><<<1, 32 * warps>>>(d, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double cyc = ms * 1e-3 * clk * 1e3;
    printf("chains %d warps %2d: %.2f cycles per DFMA warp-instr per warp, %.2f per SM-wide instr\n", CH, warps,
           cyc / ((double)iters * 16 * CH), cyc / ((double)iters * 16 * CH * warps));
}
int main() {
    double* d; cudaMalloc(&d, 4096 * 8); cudaMemset(d, 0, 4096 * 8);
    run<1>(1, d); run<2>(1, d); run<4>(1, d); run<8>(1, d);
    run<8>(2, d); run<8>(4, d); run<8>(8, d); run<8>(16, d); run<4>(32, d);
    return 0;
}
