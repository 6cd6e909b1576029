// FP64 dependent-chain latencies on the B200 (one warp): DADD, DFMA, the
// reference's mul-then-add (madd: DMUL feeding a DADD on the chain), and an
// LDS-fed madd chain.
#include <cstdio>
__global__ void lat(double* out, long long* cyc, double a, double b, int n) {
    __shared__ double sm[1024];
    for (int i = threadIdx.x; i < 1024; i += 32) sm[i] = 1e-9 * i;
    __syncwarp();
    double x = a, y = a, z = a, u = a;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = __dadd_rn(x, b);
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) y = fma(y, b, a);
    long long t2 = clock64();
    for (int i = 0; i < n; ++i) z = __dadd_rn(z, __dmul_rn(a, b + i));
    long long t3 = clock64();
    for (int i = 0; i < n; ++i) u = __dadd_rn(u, __dmul_rn(sm[(i * 7) & 1023], sm[(i * 13) & 1023]));
    long long t4 = clock64();
    out[threadIdx.x] = x + y + z + u;
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}
int main() {
    double* o; long long* c; cudaMallocManaged(&o, 256); cudaMallocManaged(&c, 64);
    lat<<<1, 32>>>(o, c, 1.0, 1e-12, 4096);
    cudaDeviceSynchronize();
    lat<<<1, 32>>>(o, c, 1.0, 1e-12, 4096);
    cudaDeviceSynchronize();
    printf("cycles/op: dadd %.1f dfma %.1f madd %.1f madd(lds) %.1f\n", c[0] / 4096.0, c[1] / 4096.0, c[2] / 4096.0, c[3] / 4096.0);
}
