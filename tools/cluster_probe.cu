// How many thread-block clusters of size C fit at once with the train
// kernel's footprint (1 CTA per SM, ~200 KB smem)? Used to pick the
// cluster size of the partial pre-reduction.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* out) {
    extern __shared__ int s[];
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    unsigned sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    if (threadIdx.x == 0) { s[0] = r; out[blockIdx.x] = (int)sm; }
}
int main() {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int* d; cudaMalloc(&d, 4096 * 4);
    for (int C : {1, 2, 4, 8, 16}) {
        cudaLaunchConfig_t cfg = {};
        cfg.blockDim = dim3(512);
        cfg.dynamicSmemBytes = 220 * 1024;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        cfg.gridDim = dim3(C * 64);
        int n = -1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (void*)k, &cfg);
        printf("cluster %2d: max active clusters %d (%d CTAs) %s\n", C, n, n * C, cudaGetErrorString(e));
        // cooperative + cluster launch of n clusters
        if (n > 0) {
            cfg.gridDim = dim3(n * C);
            at[1].id = cudaLaunchAttributeCooperative; at[1].val.cooperative = 1;
            cfg.numAttrs = 2;
            e = cudaLaunchKernelEx(&cfg, k, d);
            cudaError_t e2 = cudaDeviceSynchronize();
            printf("   cooperative+cluster launch of %d CTAs: %s / %s\n", n * C, cudaGetErrorString(e), cudaGetErrorString(e2));
        }
    }
    cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
    printf("SMs %d\n", p.multiProcessorCount);
}
