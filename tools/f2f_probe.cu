// Throughput of fp32 -> fp64 conversion (F2F.F64.F32) vs DFMA and an
// integer-op widening, per SM per clock (one CTA of 512 threads per SM,
// 8 independent chains per thread). Build: nvcc -gencode
// arch=compute_100a,code=sm_100a -O3 -o tools/f2f_probe tools/f2f_probe.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ double widen_int(float h) {  // h >= 0, normal or zero
    const uint32_t b = __float_as_uint(h);
    const uint32_t hi = b ? (b >> 3) + 0x38000000u : 0u;
    return __hiloint2double((int)hi, (int)(b << 29));
}

template <int MODE>
__global__ void __launch_bounds__(512) probe(const float* in, double* out, int iters, long long* cyc) {
    float f[8];
    double acc[8];
    for (int k = 0; k < 8; ++k) {
        f[k] = in[threadIdx.x + k];
        acc[k] = 0.0;
    }
    __syncthreads();
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (MODE == 0) acc[k] += (double)f[k];                          // F2F + DADD
            if (MODE == 1) acc[k] = fma(acc[k], 1.0000001, 0.5);            // DFMA
            if (MODE == 2) acc[k] += widen_int(f[k]);                       // integer widening + DADD
            f[k] = __uint_as_float(__float_as_uint(f[k]) ^ 1u);             // defeat hoisting
        }
    }
    __syncthreads();
    const long long t1 = clock64();
    double s = 0;
    for (int k = 0; k < 8; ++k) s += acc[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    float* in;
    double* out;
    long long* cyc;
    cudaMalloc(&in, 4096 * 4);
    cudaMalloc(&out, 148 * 512 * 8);
    cudaMalloc(&cyc, 8);
    float h[4096];
    for (int i = 0; i < 4096; ++i) h[i] = 1.0f + i * 0.001f;
    cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
    const int iters = 4096;
    const char* names[3] = {"F2F.F64.F32 + DADD", "DFMA", "integer widen + DADD"};
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            if (mode == 0) probe<0><<<148, 512>>>(in, out, iters, cyc);
            if (mode == 1) probe<1><<<148, 512>>>(in, out, iters, cyc);
            if (mode == 2) probe<2><<<148, 512>>>(in, out, iters, cyc);
            cudaDeviceSynchronize();
        }
        long long c;
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        const double ops = 512.0 * 8 * iters;
        printf("%-24s %8.1f ops/clk/SM (%lld cycles)\n", names[mode], ops / c, c);
    }
    return 0;
}
