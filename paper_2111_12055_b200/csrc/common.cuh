// common.cuh — shared device helpers for the gbxcu kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace gbxcu {

// ---------------------------------------------------------------- layout
// Policy 44 -> 64 -> 32 -> 2 (proj/include/gbx/policy.hpp:32-35), flat
// serialization offsets (proj/src/policy.cpp:226-231).
constexpr int F = 44, H1 = 64, H2 = 32, A = 2;
constexpr int OFF_W0 = 0;
constexpr int OFF_B0 = OFF_W0 + H1 * F;   // 2816
constexpr int OFF_W1 = OFF_B0 + H1;       // 2880
constexpr int OFF_B1 = OFF_W1 + H2 * H1;  // 4928
constexpr int OFF_W2 = OFF_B1 + H2;       // 4960
constexpr int OFF_B2 = OFF_W2 + A * H2;   // 5024
constexpr int NP = OFF_B2 + A;            // 5026

// --------------------------------------------------------------- SplitMix64
// proj/include/gbx/rng.hpp:11-68. The k-th output (k >= 1) of a stream
// seeded s is fin(s + k*gamma), which is what makes skip-ahead free.
constexpr uint64_t GAMMA = 0x9E3779B97F4A7C15ULL;

__host__ __device__ __forceinline__ uint64_t fin64(uint64_t x) {
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) { return fin64(x + GAMMA); }

__host__ __device__ __forceinline__ uint64_t derive_seed3(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t h = 0x8557D1C3C2DB0F5BULL;
    h = mix64(h ^ a);
    h = mix64(h ^ b);
    h = mix64(h ^ c);
    return h;
}

// k-th (1-based) raw output of SplitMix64(seed)
__host__ __device__ __forceinline__ uint64_t sm_draw(uint64_t seed, uint64_t k) {
    return fin64(seed + k * GAMMA);
}

// next_unit: (x >> 11) * 2^-53, exact
__device__ __forceinline__ double unit_of(uint64_t x) {
    return __dmul_rn(__ull2double_rn(x >> 11), 0x1.0p-53);
}
// next_signed_unit: 2u - 1 (exact)
__device__ __forceinline__ double signed_unit_of(uint64_t x) {
    return __dsub_rn(__dmul_rn(2.0, unit_of(x)), 1.0);
}
// next_below(n): Lemire multiply-shift, high 64 bits of x*n
__device__ __forceinline__ uint64_t below_of(uint64_t x, uint64_t n) { return __umul64hi(x, n); }

// ----------------------------------------------------------- exact fp64
// Reference sums are strict mul-then-add (g++ x86-64 default has no FMA).
__device__ __forceinline__ double madd_rn(double acc, double a, double b) {
    return __dadd_rn(acc, __dmul_rn(a, b));
}

__device__ __forceinline__ double clampp(double p) {
    const double lo = 1e-7, hi = 1.0 - 1e-7;
    return p < lo ? lo : (hi < p ? hi : p);
}

// ------------------------------------------------------------ grid barrier
// Monotonic arrival counter in global memory; all CTAs of a cooperative
// launch call it the same number of times. `target` is carried by the caller
// (incremented by gridDim.x per barrier).
__device__ __forceinline__ void grid_barrier(unsigned int* counter, unsigned int& target) {
    __syncthreads();
    target += gridDim.x;
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(counter, 1u);
        unsigned int v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
        } while ((int)(v - target) < 0);
    }
    __syncthreads();
}

}  // namespace gbxcu
