// tools/peaks.cu — measured pipe peaks for the roofline denominators that
// MEASURED_PEAKS.json does not carry (it has HBM and bf16 tensor only):
// dependent-free DFMA / FFMA throughput over all SMs. Used by bench.py only.
#include <cuda_runtime.h>
#include <stdint.h>

template <typename T>
__global__ void fma_peak_kernel(T* out, int iters, T a, T b) {
    T x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5,
      x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            x0 = x0 * a + b; x1 = x1 * a + b; x2 = x2 * a + b; x3 = x3 * a + b;
            x4 = x4 * a + b; x5 = x5 * a + b; x6 = x6 * a + b; x7 = x7 * a + b;
        }
    }
    T s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (s == (T)-12345.0) out[0] = s;
}

// FP64 tensor-core (DMMA 8x8x4) throughput: 8 independent accumulator pairs per warp.
__global__ void dmma_peak_kernel(double* out, int iters) {
    double a = 0.5 + threadIdx.x * 1e-3, b = 0.25;
    double c[8][2];
#pragma unroll
    for (int q = 0; q < 8; ++q) c[q][0] = c[q][1] = q;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int q = 0; q < 8; ++q)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1},{%2},{%3},{%0,%1};"
                         : "+d"(c[q][0]), "+d"(c[q][1]) : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += c[q][0] + c[q][1];
    if (s == -12345.0) out[0] = s;
}

static double run_dmma(int device, int iters) {
    cudaSetDevice(device);
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, device);
    double* out;
    cudaMalloc(&out, sizeof(double));
    const int blocks = prop.multiProcessorCount * 4, threads = 256;
    dmma_peak_kernel<<<blocks, threads>>>(out, 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double best = 0;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        dmma_peak_kernel<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        // 8x8x4 = 256 FMA = 512 FLOP per warp-instruction
        const double flops = 512.0 * 8 * (double)iters * blocks * (threads / 32);
        best = best > flops / (ms * 1e-3) ? best : flops / (ms * 1e-3);
    }
    cudaFree(out);
    return best / 1e12;
}

template <typename T>
static double run(int device, int iters) {
    cudaSetDevice(device);
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, device);
    T* out;
    cudaMalloc(&out, sizeof(T));
    const int blocks = prop.multiProcessorCount * 8, threads = 256;
    fma_peak_kernel<T><<<blocks, threads>>>(out, 16, (T)0.999, (T)0.001);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double best = 0;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        fma_peak_kernel<T><<<blocks, threads>>>(out, iters, (T)0.999, (T)0.001);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
        best = best > flops / (ms * 1e-3) ? best : flops / (ms * 1e-3);
    }
    cudaFree(out);
    return best / 1e12;
}

extern "C" double peak_fp64_tflops(int device) { return run<double>(device, 4096); }
extern "C" double peak_fp32_tflops(int device) { return run<float>(device, 16384); }
extern "C" double peak_fp64_tensor_tflops(int device) { return run_dmma(device, 8192); }

// DMMA dependent-chain latency: one warp, one accumulator chain.
__global__ void dmma_latency_kernel(double* out, int iters, long long* cycles) {
    double a = 0.5 + threadIdx.x * 1e-3, b = 0.25, c0 = 0, c1 = 0;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1},{%2},{%3},{%0,%1};"
                     : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
    const long long t1 = clock64();
    if (threadIdx.x == 0) *cycles = t1 - t0;
    if (c0 + c1 == -12345.0) out[0] = c0;
}

extern "C" double dmma_latency_cycles(int device) {
    cudaSetDevice(device);
    double* out;
    long long* cyc;
    cudaMalloc(&out, sizeof(double));
    cudaMalloc(&cyc, sizeof(long long));
    dmma_latency_kernel<<<1, 32>>>(out, 1000, cyc);
    dmma_latency_kernel<<<1, 32>>>(out, 1000, cyc);
    long long h = 0;
    cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    cudaFree(out);
    cudaFree(cyc);
    return h / 1000.0;
}
