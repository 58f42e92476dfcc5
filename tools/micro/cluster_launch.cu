// Fixed cost of a thread-block-cluster launch shaped like the chunk carry
// (7 clusters, 1024 threads per CTA, ~135 KB dynamic shared memory, two
// cluster barriers): back-to-back launches, time per launch.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/cluster_launch tools/micro/cluster_launch.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

template <bool CL>
__global__ void __launch_bounds__(1024, 1) k(int nsync, double* out) {
    extern __shared__ double sm[];
    if (threadIdx.x < 512) sm[threadIdx.x] = 0.0;
    if (CL) {
        cg::cluster_group cl = cg::this_cluster();
        for (int i = 0; i < nsync; ++i) cl.sync();
    } else {
        for (int i = 0; i < nsync; ++i) __syncthreads();
    }
    if (out && threadIdx.x == 0 && blockIdx.x == 0) out[0] = sm[0];
}

static float run(int cs, int clusters, int threads, int smem, int nsync) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(cs * clusters); cfg.blockDim = dim3(threads); cfg.dynamicSmemBytes = smem;
    cfg.attrs = at; cfg.numAttrs = cs > 1 ? 1 : 0;
    auto f = cs > 1 ? k<true> : k<false>;
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (cs > 8) cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int i = 0; i < 10; ++i) cudaLaunchKernelEx(&cfg, f, nsync, (double*)nullptr);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int i = 0; i < 200; ++i) cudaLaunchKernelEx(&cfg, f, nsync, (double*)nullptr);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error: %s\n", cudaGetErrorString(e));
    return ms * 1000.f / 200.f;
}

int main() {
    const int smem = 135 * 1024;
    printf("cs clusters threads smem nsync us/launch\n");
    for (int cs : {1, 2, 4, 8, 16})
        for (int th : {256, 1024})
            for (int sm : {8 * 1024, smem})
                for (int ns : {0, 2})
                    printf("%2d %3d %4d %6d %d %7.2f\n", cs, 112 / cs, th, sm, ns, run(cs, 112 / cs, th, sm, ns));
    return 0;
}
