// tools/tc_probe.cu — hardware probe of the tcgen05 TF32 path used by the
// product kernels: one CTA computes D[128][N] = A[128][K] . B[N][K]^T through
// shared-memory descriptors, TMEM accumulation and tcgen05.ld. Used to validate
// descriptor encodings and to measure TF32 operand rounding / accumulation
// error against fp64 (tools/tc_probe.py). Not part of the product.
#include <cuda_runtime.h>
#include <stdint.h>
#include "../paper_2111_12055_b200/csrc/tc_util.cuh"

using namespace gbxcu::tc;

template <int N>
__global__ void __launch_bounds__(128) tc_probe_kernel(const float* A, const float* B, float* D, int K) {
    extern __shared__ __align__(1024) unsigned char smem[];
    float* As = reinterpret_cast<float*>(smem);
    float* Bs = As + 128 * K;
    __shared__ uint64_t mbar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 128 * K; i += 128) {
        const int r = i / K, k = i % K;
        As[canon_off(r, k, 128) / 4] = A[i];
    }
    for (int i = tid; i < N * K; i += 128) {
        const int r = i / K, k = i % K;
        Bs[canon_off(r, k, N) / 4] = B[i];
    }
    if (w == 0) tmem_alloc(&tbase, N < 32 ? 32 : N);
    if (tid == 0) { mbar_init(&mbar, 1); fence_mbar_init(); }
    fence_async_smem();
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t t0 = tbase;
    if (tid == 0) {
        for (int s = 0; s < K / 8; ++s) {
            const uint64_t ad = smem_desc(smem_u32(As) + 2 * s * 128 * 16, 128 * 16, 128);
            const uint64_t bd = smem_desc(smem_u32(Bs) + 2 * s * N * 16, N * 16, 128);
            mma_tf32(t0, ad, bd, idesc_tf32(128, N), s > 0);
        }
        commit_to(&mbar);
    }
    mbar_wait(&mbar, 0);
    fence_after_sync();
    for (int c0 = 0; c0 < N; c0 += 16) {
        float v[16];
        tmem_ld16(t0 + ((uint32_t)(32 * w) << 16) + c0, v);
        tmem_ld_wait();
        for (int i = 0; i < 16; ++i) D[(32 * w + lane) * N + c0 + i] = v[i];
    }
    fence_before_sync();
    __syncthreads();
    if (w == 0) tmem_dealloc(t0, N < 32 ? 32 : N);
}

extern "C" int tc_probe(const float* hA, const float* hB, float* hD, int N, int K) {
    float *A, *B, *D;
    cudaMalloc(&A, 128 * K * 4); cudaMalloc(&B, N * K * 4); cudaMalloc(&D, 128 * N * 4);
    cudaMemcpy(A, hA, 128 * K * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(B, hB, N * K * 4, cudaMemcpyHostToDevice);
    const int smem = (128 + N) * K * 4;
    if (N == 64) {
        cudaFuncSetAttribute(tc_probe_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        tc_probe_kernel<64><<<1, 128, smem>>>(A, B, D, K);
    } else if (N == 32) {
        cudaFuncSetAttribute(tc_probe_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        tc_probe_kernel<32><<<1, 128, smem>>>(A, B, D, K);
    } else if (N == 256) {
        cudaFuncSetAttribute(tc_probe_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        tc_probe_kernel<256><<<1, 128, smem>>>(A, B, D, K);
    } else return -1;
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(hD, D, 128 * N * 4, cudaMemcpyDeviceToHost);
    cudaFree(A); cudaFree(B); cudaFree(D);
    return (int)e;
}
