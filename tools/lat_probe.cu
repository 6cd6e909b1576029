// Latency probe: dependent DADD / DFMA / FADD chains and an LDS->DADD chain (one warp).
#include <cstdio>
__global__ void k(double* out, long long* cyc, int iters, double x) {
    __shared__ double sm[64];
    sm[threadIdx.x] = x + threadIdx.x;
    __syncwarp();
    double a = x, b = x * 0.5;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) a = __dadd_rn(a, b);
    long long t1 = clock64();
    for (int i = 0; i < iters; ++i) a = fma(a, b, 1e-300);
    long long t2 = clock64();
    float f = (float)a, g = 0.5f;
    for (int i = 0; i < iters; ++i) f = __fadd_rn(f, g);
    long long t3 = clock64();
    int idx = threadIdx.x & 31;
    for (int i = 0; i < iters; ++i) { a = __dadd_rn(a, sm[idx]); idx = (idx + 1) & 31; }
    long long t4 = clock64();
    for (int i = 0; i < iters; ++i) a = __ddiv_rn(b, a + 1.0);
    long long t5 = clock64();
    out[threadIdx.x] = a + f;
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; }
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 64 * 8); cudaMallocManaged(&c, 64);
    const int it = 4096;
    k<<<1, 32>>>(o, c, it, 1.0); cudaDeviceSynchronize();
    k<<<1, 32>>>(o, c, it, 1.0); cudaDeviceSynchronize();
    printf("cycles per dependent op: DADD %.1f DFMA %.1f FADD %.1f LDS+DADD %.1f DDIV %.1f\n",
           c[0] / (double)it, c[1] / (double)it, c[2] / (double)it, c[3] / (double)it, c[4] / (double)it);
}
