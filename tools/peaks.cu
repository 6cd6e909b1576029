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
