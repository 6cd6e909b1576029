// Do the FP64 tensor path (DMMA m8n8k4) and the FP64 FMA pipe (DFMA) run
// concurrently on B200? One CTA of 512 threads per SM; warps 0..7 issue DMMA,
// warps 8..15 DFMA (mode 2), or all warps one kind (modes 0, 1). Reports
// FLOP/clk/SM. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o
// tools/fp64_mix tools/fp64_mix.cu
#include <cstdio>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

constexpr int DF = 4;
template <int MODE>
__global__ void __launch_bounds__(512) probe(double* out, int iters, long long* cyc) {
    const int w = threadIdx.x >> 5;
    const bool do_mma = MODE == 0 || (MODE == 2 && w < 8);
    double acc[8][2];
    for (int k = 0; k < 8; ++k) acc[k][0] = acc[k][1] = 0.001 * threadIdx.x + k;
    const double a = 1.0000001, b = 0.9999999;
    __syncthreads();
    const long long t0 = clock64();
    if (do_mma) {
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int k = 0; k < 8; ++k) dmma(acc[k], a, b);
        }
    } else {
        const int n = MODE == 2 ? iters * DF : iters;  // (mode 2: DF x the iterations, to balance the halves)
        for (int i = 0; i < n; ++i) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                acc[k][0] = fma(acc[k][0], a, b);
                acc[k][1] = fma(acc[k][1], b, a);
            }
        }
    }
    __syncthreads();
    const long long t1 = clock64();
    double s = 0;
    for (int k = 0; k < 8; ++k) s += acc[k][0] + acc[k][1];
    out[blockIdx.x * 512 + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 148 * 512 * 8);
    cudaMalloc(&cyc, 8);
    const int iters = 2048;
    const char* names[3] = {"DMMA only (16 warps)", "DFMA only (16 warps)", "8 warps DMMA + 8 warps DFMA"};
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            if (mode == 0) probe<0><<<148, 512>>>(out, iters, cyc);
            if (mode == 1) probe<1><<<148, 512>>>(out, iters, cyc);
            if (mode == 2) probe<2><<<148, 512>>>(out, iters, cyc);
            cudaDeviceSynchronize();
        }
        long long c;
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        // per warp per iteration: 8 DMMA x 512 FLOP, or 32 lanes x 16 DFMA x 2 FLOP = 1024
        double flop;
        if (mode == 0) flop = 16.0 * iters * 8 * 512;
        else if (mode == 1) flop = 16.0 * iters * 1024;
        else flop = 8.0 * iters * 8 * 512 + 8.0 * iters * DF * 1024;
        printf("%-30s %7.1f FLOP/clk/SM  (%lld cycles)\n", names[mode], flop / c, c);
    }
    return 0;
}
