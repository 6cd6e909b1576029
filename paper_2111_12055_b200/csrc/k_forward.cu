// k_forward.cu — batched policy inference (K2) for sm_100a.
//
// Replaces PolicyNet::forward / select_greedy / select_sample
// (proj/src/policy.cpp:29-55,141-148,339-347) and the collection-mode draw of
// run_iteration (proj/src/tuner.cpp:183-196).
//
// Two paths:
//   * fwd_fast_kernel  — one thread per state, fp32 FFMA, weights in shared
//     memory (broadcast LDS.128), layers 1 and 2 interleaved so h1 never
//     materialises. Each state carries a rigorous forward error bound on its
//     logit difference (see guard_threshold); states whose margin is inside
//     the bound are appended to a re-check list.
//   * fwd_exact_kernel — one thread per state, fp64 in the reference's exact
//     summation order (bias first, ascending index; layer-1 products are exact
//     in fp64 so DFMA is used there, layers 2-3 use mul-then-add rounding).
//     Runs either over all states (EXACT mode) or over the re-check list.
#include <cstddef>

#include "common.cuh"
#include "kernels.h"

namespace gbxcu {

// ------------------------------------------------------------ policy init
// PolicyNet::init (proj/src/policy.cpp:128-139).
__global__ void policy_init_kernel(uint64_t seed, float* __restrict__ params) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= NP) return;
    int l, k;
    if (t < OFF_B0) { l = 0; k = t - OFF_W0; }
    else if (t < OFF_W1) { params[t] = 0.f; return; }
    else if (t < OFF_B1) { l = 1; k = t - OFF_W1; }
    else if (t < OFF_W2) { params[t] = 0.f; return; }
    else if (t < OFF_B2) { l = 2; k = t - OFF_W2; }
    else { params[t] = 0.f; return; }
    const int dims[4] = {F, H1, H2, A};
    const double bound = sqrt(6.0 / (double)(dims[l] + dims[l + 1]));
    const uint64_t s = derive_seed3(seed, 0x1A17u, (uint64_t)l);
    const double u = signed_unit_of(sm_draw(s, (uint64_t)k + 1));
    params[t] = __double2float_rn(__dmul_rn(u, bound));
}

// Stage the 5,026 fp32 parameters into shared memory with ONE memory round
// trip (16-B cp.async chunks, all in flight at once); each kernel then builds
// its own layout from the staged copy. (A strided per-element loop costs one
// L2 round trip per iteration: ~20 of them, ~15 us, at every launch.)
__device__ void stage_params(float* raw, const float* __restrict__ p) {
    if ((reinterpret_cast<uintptr_t>(p) & 15u) == 0) {
        for (int c = threadIdx.x; c < NP / 4; c += blockDim.x) {
            const unsigned d = (unsigned)__cvta_generic_to_shared(raw + 4 * c);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(p + 4 * c) : "memory");
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
        for (int t = (NP / 4) * 4 + threadIdx.x; t < NP; t += blockDim.x) raw[t] = __ldg(p + t);
        asm volatile("cp.async.wait_all;\n" ::: "memory");
    } else {
        for (int t = threadIdx.x; t < NP; t += blockDim.x) raw[t] = __ldg(p + t);
    }
    __syncthreads();
}

// --------------------------------------------------------------- fast path
constexpr int FAST_ROWS = 64;  // states per warp per iteration (two per lane)
// Weights are laid out for packed FFMA2 (two fp32 FMAs per instruction, each
// with its own single rounding — numerically identical to two FFMAs):
//   w0p [j/2][i][2] pairs rows j, j+1 of W0, so one FFMA2 advances z_j, z_j+1;
//   w1t [j][k]      consecutive k pairs advance acc2[k], acc2[k+1];
//   w2p [k][2]      advances both logits.
struct FastSmem {
    __align__(16) float xs[FWD_BLOCK / 32][2][FAST_ROWS * F];  // per-warp double-buffered staging
    float w0[H1 * F];   // w0p: [j/2][i][j&1]
    float w1t[H1 * H2]; // [j][k] = w1[k][j]
    float w2[A * H2];   // w2p: [k][a]
    float b0[H1];
    float b1[H2];
    float b2[A];
    float stats[12];    // R0,B0,R1,B1,R2,B2,Rd,W0max,W1max
};
static_assert(offsetof(FastSmem, w0) % 16 == 0 && offsetof(FastSmem, w1t) % 16 == 0, "align");

// Per-net constants of the guard: R_l = max_row ||w_row||_1, B_l = max |b|,
// Rd = ||w2[1] - w2[0]||_1. Computed in fp64 and rounded up so the fp32 bound
// stays an upper bound. `raw` = the staged parameters (S.xs, free until the
// first feature tile is staged).
__device__ void load_fast_weights(FastSmem& S, float* raw, const float* __restrict__ p) {
    stage_params(raw, p);
    for (int t = threadIdx.x; t < H1 * F; t += blockDim.x) {
        const int j = t / F, i = t - j * F;
        S.w0[(j >> 1) * (2 * F) + 2 * i + (j & 1)] = raw[OFF_W0 + t];
    }
    for (int t = threadIdx.x; t < H1 * H2; t += blockDim.x) {
        const int k = t / H1, j = t % H1;
        S.w1t[j * H2 + k] = raw[OFF_W1 + t];
    }
    for (int t = threadIdx.x; t < A * H2; t += blockDim.x) S.w2[(t % H2) * A + t / H2] = raw[OFF_W2 + t];
    for (int t = threadIdx.x; t < H1; t += blockDim.x) S.b0[t] = raw[OFF_B0 + t];
    for (int t = threadIdx.x; t < H2; t += blockDim.x) S.b1[t] = raw[OFF_B1 + t];
    if (threadIdx.x < A) S.b2[threadIdx.x] = raw[OFF_B2 + threadIdx.x];
    __syncthreads();
    // per-row / per-column norms in parallel (fp64), then one warp reduces
    double* nrm = reinterpret_cast<double*>(raw);  // [0,64) r0 rows, [64,96) r1 cols, [96,98) r2, [128,160) rd
    const int t = threadIdx.x;
    if (t < H1) {
        double s = 0;
        for (int i = 0; i < F; ++i) s += fabs((double)S.w0[(t >> 1) * (2 * F) + 2 * i + (t & 1)]);
        nrm[t] = s;
    } else if (t < H1 + H2) {
        double s = 0;
        for (int j = 0; j < H1; ++j) s += fabs((double)S.w1t[j * H2 + (t - H1)]);
        nrm[t] = s;
    } else if (t < H1 + H2 + A) {
        double s = 0;
        for (int k = 0; k < H2; ++k) s += fabs((double)S.w2[k * A + (t - H1 - H2)]);
        nrm[t] = s;
    } else if (t >= 128 && t < 128 + H2) {
        const int k = t - 128;
        nrm[t] = fabs((double)S.w2[k * A + 1] - (double)S.w2[k * A]);
    } else if (t >= 160 && t < 160 + H1) {
        // per-unit max |w0[j][i]| (slot 160+j) and max |w1[k][j]| over k (slot 224+j)
        const int j = t - 160;
        double m0 = 0, m1 = 0;
        for (int i = 0; i < F; ++i) m0 = fmax(m0, fabs((double)S.w0[(j >> 1) * (2 * F) + 2 * i + (j & 1)]));
        for (int k = 0; k < H2; ++k) m1 = fmax(m1, fabs((double)S.w1t[j * H2 + k]));
        nrm[t] = m0;
        nrm[t + H1] = m1;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        double r0 = fmax(nrm[lane], nrm[lane + 32]);
        double bb0 = fmax(fabs((double)S.b0[lane]), fabs((double)S.b0[lane + 32]));
        double r1 = nrm[H1 + lane], bb1 = fabs((double)S.b1[lane]);
        double r2 = lane < A ? nrm[H1 + H2 + lane] : 0.0;
        double bb2 = lane < A ? fabs((double)S.b2[lane]) : 0.0;
        double rd = nrm[128 + lane];
        double wm0 = fmax(nrm[160 + lane], nrm[192 + lane]);
        double wm1 = fmax(nrm[224 + lane], nrm[256 + lane]);
        for (int o = 16; o > 0; o >>= 1) {
            r0 = fmax(r0, __shfl_xor_sync(0xffffffffu, r0, o));
            bb0 = fmax(bb0, __shfl_xor_sync(0xffffffffu, bb0, o));
            r1 = fmax(r1, __shfl_xor_sync(0xffffffffu, r1, o));
            bb1 = fmax(bb1, __shfl_xor_sync(0xffffffffu, bb1, o));
            r2 = fmax(r2, __shfl_xor_sync(0xffffffffu, r2, o));
            bb2 = fmax(bb2, __shfl_xor_sync(0xffffffffu, bb2, o));
            rd += __shfl_xor_sync(0xffffffffu, rd, o);
            wm0 = fmax(wm0, __shfl_xor_sync(0xffffffffu, wm0, o));
            wm1 = fmax(wm1, __shfl_xor_sync(0xffffffffu, wm1, o));
        }
        if (lane == 0) {
            // 1.0001 absorbs the rounding of the fp64 row sums themselves
            S.stats[0] = __double2float_ru(r0 * 1.0001);
            S.stats[1] = __double2float_ru(bb0);
            S.stats[2] = __double2float_ru(r1 * 1.0001);
            S.stats[3] = __double2float_ru(bb1);
            S.stats[4] = __double2float_ru(r2 * 1.0001);
            S.stats[5] = __double2float_ru(bb2);
            S.stats[6] = __double2float_ru(rd * 1.0001);
            S.stats[7] = __double2float_ru(wm0);
            S.stats[8] = __double2float_ru(wm1);
        }
    }
    __syncthreads();
}

// Forward error bound on |(l1-l0)_fp32 - (l1-l0)_exact| (Higham-style
// recursive-summation bounds for FMA chains, u = 2^-24, g(n) = n u (1 + 1e-4)):
//   D1 = g(14)(B0 + min(R0 X, W0 X1))  X = max_i |x_i|, X1 = sum_i |x_i|,
//                                 W0 = max |w0| (either product bounds
//                                 sum_i |w_ji||x_i|); layer 1 runs 4 chains of
//                                 <= 12 terms (bias in the first) + 2 levels
//                                 of adds: 14 roundings per element at most
//   D2 = g(65)(B1 + min(R1 H1, W1 H1s)) + R1 D1   H1 = max_j h1_j, H1s = sum_j h1_j
//   e3 = 2 g(33)(B2 + R2 H2) + Rd D2   H2 = max_k h2_k; Rd = ||w2[1] - w2[0]||_1
//        (each logit's own chain rounding, plus the difference's sensitivity
//        to the h2 errors, which relu does not amplify)
//   margin = 1.01 e3 (+ slack for the fp64 reference's own rounding, the
//   final fp32 subtraction and this bound's evaluation).
__device__ __forceinline__ float guard_threshold(const float* st, float X, float X1, float Hm1,
                                                 float H1s, float Hm2) {
    const float u = 5.9604645e-8f;  // 2^-24
    const float g14 = 14.f * u * 1.0001f, g65 = 65.f * u * 1.0001f, g33 = 33.f * u * 1.0001f;
    // sum_i |w_ji| |x_i| <= min(R0 max|x|, max|w0| sum|x|); likewise for layer 2
    const float D1 = g14 * (st[1] + fminf(st[0] * X, st[7] * X1));
    const float D2 = g65 * (st[3] + fminf(st[2] * Hm1, st[8] * H1s)) + st[2] * D1;
    const float e3 = 2.f * g33 * (st[5] + st[4] * Hm2) + st[6] * D2;
    return 1.02f * e3 + 1e-30f;
}

// Per-state tail of the fast path: guard, fp32 softmax, action (greedy or
// collection draw), re-check list, outputs.
__device__ __forceinline__ void fast_finish(const FastSmem& S, size_t s, float l0, float l1,
                                            float X, float X1, float hm1, float h1s, float hm2,
                                            bool finite,
                                            double* __restrict__ probs, uint8_t* __restrict__ actions,
                                            const uint64_t* __restrict__ seg_off, size_t nseg,
                                            const uint64_t* __restrict__ seg_seed, double eps,
                                            uint32_t* __restrict__ recheck,
                                            unsigned int* __restrict__ n_recheck,
                                            unsigned int* __restrict__ flags, int mode) {
    if (!finite) {
        atomicOr(flags, 1u);
        return;
    }
    const float T = guard_threshold(S.stats, X, X1, hm1, h1s, hm2);
    const float d = l1 - l0;
    // fp32 softmax (max-subtracted like the reference)
    const float m = fmaxf(l0, l1);
    const float e0 = expf(l0 - m), e1 = expf(l1 - m);
    const float p0 = e0 / (e0 + e1);
    bool ambiguous;
    uint8_t act;
    if (mode & 8) {
        // select_sample over one stream: state s takes draw s + 1 of seg_seed[0]
        const double ua = unit_of(sm_draw(seg_seed[0], (uint64_t)s + 1));
        const double tol = 0.25 * (double)T + 16.0 * 5.9604645e-8;
        ambiguous = fabs(ua - (double)p0) <= tol;
        act = ua < (double)p0 ? 0 : 1;
    } else if (mode & 4) {
        // collection: find this state's segment and its two draws
        size_t lo = 0, hi = nseg;  // seg_off[lo] <= s < seg_off[hi]
        while (hi - lo > 1) {
            const size_t mid = (lo + hi) >> 1;
            if (seg_off[mid] <= s) lo = mid; else hi = mid;
        }
        const uint64_t j = s - seg_off[lo];
        const uint64_t seed = seg_seed[lo];
        const double ue = unit_of(sm_draw(seed, 2 * j + 1));
        const double ua = unit_of(sm_draw(seed, 2 * j + 2));
        if (ue < eps) {
            act = ua < 0.5 ? 0 : 1;
            ambiguous = false;
        } else {
            // |p0_fp32 - p0_exact| <= |dp0/dd| * 2D3 + fp32 rounding of exp/div
            //                     <= 0.25 * T + 16 u
            const double tol = 0.25 * (double)T + 16.0 * 5.9604645e-8;
            ambiguous = fabs(ua - (double)p0) <= tol;
            act = ua < (double)p0 ? 0 : 1;
        }
    } else {
        ambiguous = !(fabsf(d) > T);
        act = d > 0.f ? 1 : 0;
    }
    if (ambiguous) {
        const unsigned int slot = atomicAdd(n_recheck, 1u);
        recheck[slot] = (uint32_t)s;
    }
    if (mode & 2) actions[s] = act;
    if (mode & 1) {
        probs[2 * s] = (double)p0;
        probs[2 * s + 1] = (double)(e1 / (e0 + e1));
    }
}

// Loads one staged row into registers; returns max |x| and finiteness.
__device__ __forceinline__ void fast_row(const float* xs, int r, float (&x)[F], float& X, float& X1,
                                         bool& finite) {
    const float4* row = reinterpret_cast<const float4*>(xs + r * F);
#pragma unroll
    for (int q = 0; q < F / 4; ++q) {
        const float4 v = row[q];
        x[4 * q] = v.x; x[4 * q + 1] = v.y; x[4 * q + 2] = v.z; x[4 * q + 3] = v.w;
    }
    X = 0.f;
    X1 = 0.f;
    finite = true;
#pragma unroll
    for (int i = 0; i < F; ++i) {
        finite &= isfinite(x[i]);
        X = fmaxf(X, fabsf(x[i]));
        X1 += fabsf(x[i]);
    }
}

// mode bits: 1 = write probs, 2 = write actions, 4 = collect (sampled) mode.
// Each lane evaluates two states (rows lane and lane + 32 of the warp's
// 64-row tile): every weight read from shared memory feeds two packed FFMA2s,
// which keeps the shared-memory instruction rate below the FMA pipe's.
__global__ void __launch_bounds__(FWD_BLOCK, 1)
fwd_fast_kernel(const float* __restrict__ params, const float* __restrict__ feat, size_t n,
                double* __restrict__ probs, uint8_t* __restrict__ actions,
                const uint64_t* __restrict__ seg_off, size_t nseg,
                const uint64_t* __restrict__ seg_seed, double eps,
                uint32_t* __restrict__ recheck, unsigned int* __restrict__ n_recheck,
                unsigned int* __restrict__ flags, int mode) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    FastSmem& S = *reinterpret_cast<FastSmem*>(smem_raw);
    load_fast_weights(S, &S.xs[0][0][0], params);

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const size_t n_warps_total = (size_t)gridDim.x * (FWD_BLOCK / 32);
    // rows of this warp's next pass stream in (cp.async) while the current one computes
    auto stage = [&](size_t b, int buf) {
        if (b < n) {
            const int nvec = (int)min((size_t)FAST_ROWS, n - b) * (F / 4);
            const float4* src = reinterpret_cast<const float4*>(feat + b * F);
            float4* dst = reinterpret_cast<float4*>(S.xs[warp][buf]);
            for (int v = lane; v < nvec; v += 32) {
                const unsigned d = (unsigned)__cvta_generic_to_shared(dst + v);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src + v) : "memory");
            }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    size_t base = ((size_t)blockIdx.x * (FWD_BLOCK / 32) + warp) * FAST_ROWS;
    int buf = 0;
    stage(base, 0);
    for (; base < n; base += n_warps_total * FAST_ROWS, buf ^= 1) {
        stage(base + n_warps_total * FAST_ROWS, buf ^ 1);
        asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        __syncwarp();
        const float* xs = S.xs[warp][buf];
        const size_t rows = min((size_t)FAST_ROWS, n - base);
        const bool act0 = lane < (int)rows, act1 = lane + 32 < (int)rows;

        float xa[F], xb[F];
        float Xa, Xb, X1a, X1b;
        bool fa, fb;
        fast_row(xs, act0 ? lane : 0, xa, Xa, X1a, fa);
        fast_row(xs, act1 ? lane + 32 : 0, xb, Xb, X1b, fb);
        __syncwarp();  // the buffer is refilled two passes later

        // ---- layers 1+2 interleaved: acc2[k] += w1[k][j] * relu(z1_j), packed FFMA2
        float2 ca[H2 / 2], cb[H2 / 2];
#pragma unroll
        for (int q = 0; q < H2 / 2; ++q) ca[q] = cb[q] = make_float2(S.b1[2 * q], S.b1[2 * q + 1]);
        float hma = 0.f, hmb = 0.f, hsa = 0.f, hsb = 0.f;
#pragma unroll 2
        for (int jp = 0; jp < H1 / 2; ++jp) {
            const float4* wr = reinterpret_cast<const float4*>(S.w0 + jp * (2 * F));
            // four partial chains per z (inputs i mod 4): ILP and a 4x shorter
            // rounding chain; the guard's bound (g(14)) holds for this order
            float2 za = make_float2(S.b0[2 * jp], S.b0[2 * jp + 1]), zb = za;
            float2 za2 = make_float2(0.f, 0.f), zb2 = za2, za3 = za2, zb3 = za2, za4 = za2, zb4 = za2;
#pragma unroll
            for (int q = 0; q < F / 2; q += 2) {
                const float4 w = wr[q], v = wr[q + 1];
                const float2 w01 = make_float2(w.x, w.y), w23 = make_float2(w.z, w.w);
                const float2 v01 = make_float2(v.x, v.y), v23 = make_float2(v.z, v.w);
                za = __ffma2_rn(w01, make_float2(xa[2 * q], xa[2 * q]), za);
                zb = __ffma2_rn(w01, make_float2(xb[2 * q], xb[2 * q]), zb);
                za2 = __ffma2_rn(w23, make_float2(xa[2 * q + 1], xa[2 * q + 1]), za2);
                zb2 = __ffma2_rn(w23, make_float2(xb[2 * q + 1], xb[2 * q + 1]), zb2);
                za3 = __ffma2_rn(v01, make_float2(xa[2 * q + 2], xa[2 * q + 2]), za3);
                zb3 = __ffma2_rn(v01, make_float2(xb[2 * q + 2], xb[2 * q + 2]), zb3);
                za4 = __ffma2_rn(v23, make_float2(xa[2 * q + 3], xa[2 * q + 3]), za4);
                zb4 = __ffma2_rn(v23, make_float2(xb[2 * q + 3], xb[2 * q + 3]), zb4);
            }
            za = make_float2((za.x + za3.x) + (za2.x + za4.x), (za.y + za3.y) + (za2.y + za4.y));
            zb = make_float2((zb.x + zb3.x) + (zb2.x + zb4.x), (zb.y + zb3.y) + (zb2.y + zb4.y));
            const float hA0 = za.x > 0.f ? za.x : 0.f, hA1 = za.y > 0.f ? za.y : 0.f;
            const float hB0 = zb.x > 0.f ? zb.x : 0.f, hB1 = zb.y > 0.f ? zb.y : 0.f;
            hma = fmaxf(hma, fmaxf(hA0, hA1));
            hmb = fmaxf(hmb, fmaxf(hB0, hB1));
            hsa += hA0 + hA1;
            hsb += hB0 + hB1;
            const float4* w1a = reinterpret_cast<const float4*>(S.w1t + (2 * jp) * H2);
            const float4* w1b = reinterpret_cast<const float4*>(S.w1t + (2 * jp + 1) * H2);
#pragma unroll
            for (int q = 0; q < H2 / 4; ++q) {
                const float4 w = w1a[q];
                const float2 w01 = make_float2(w.x, w.y), w23 = make_float2(w.z, w.w);
                ca[2 * q] = __ffma2_rn(w01, make_float2(hA0, hA0), ca[2 * q]);
                cb[2 * q] = __ffma2_rn(w01, make_float2(hB0, hB0), cb[2 * q]);
                ca[2 * q + 1] = __ffma2_rn(w23, make_float2(hA0, hA0), ca[2 * q + 1]);
                cb[2 * q + 1] = __ffma2_rn(w23, make_float2(hB0, hB0), cb[2 * q + 1]);
            }
#pragma unroll
            for (int q = 0; q < H2 / 4; ++q) {
                const float4 w = w1b[q];
                const float2 w01 = make_float2(w.x, w.y), w23 = make_float2(w.z, w.w);
                ca[2 * q] = __ffma2_rn(w01, make_float2(hA1, hA1), ca[2 * q]);
                cb[2 * q] = __ffma2_rn(w01, make_float2(hB1, hB1), cb[2 * q]);
                ca[2 * q + 1] = __ffma2_rn(w23, make_float2(hA1, hA1), ca[2 * q + 1]);
                cb[2 * q + 1] = __ffma2_rn(w23, make_float2(hB1, hB1), cb[2 * q + 1]);
            }
        }
        float2 la = make_float2(S.b2[0], S.b2[1]), lb = la;
        float h2a = 0.f, h2b = 0.f;
        const float2* w2p = reinterpret_cast<const float2*>(S.w2);
#pragma unroll
        for (int q = 0; q < H2 / 2; ++q) {
            const float a0 = ca[q].x > 0.f ? ca[q].x : 0.f, a1 = ca[q].y > 0.f ? ca[q].y : 0.f;
            const float b0 = cb[q].x > 0.f ? cb[q].x : 0.f, b1 = cb[q].y > 0.f ? cb[q].y : 0.f;
            h2a = fmaxf(h2a, fmaxf(a0, a1));
            h2b = fmaxf(h2b, fmaxf(b0, b1));
            la = __ffma2_rn(w2p[2 * q], make_float2(a0, a0), la);
            lb = __ffma2_rn(w2p[2 * q], make_float2(b0, b0), lb);
            la = __ffma2_rn(w2p[2 * q + 1], make_float2(a1, a1), la);
            lb = __ffma2_rn(w2p[2 * q + 1], make_float2(b1, b1), lb);
        }
        if (act0)
            fast_finish(S, base + lane, la.x, la.y, Xa, X1a, hma, hsa, h2a, fa, probs, actions, seg_off, nseg,
                        seg_seed, eps, recheck, n_recheck, flags, mode);
        if (act1)
            fast_finish(S, base + 32 + lane, lb.x, lb.y, Xb, X1b, hmb, hsb, h2b, fb, probs, actions, seg_off,
                        nseg, seg_seed, eps, recheck, n_recheck, flags, mode);
    }
}

// -------------------------------------------------------------- exact path
struct ExactSmem {
    double w0[H1 * F];   // [j][i]
    double w1t[H1 * H2]; // [j][k]
    double w2[A * H2];
    double b0[H1];
    double b1[H2];
    double b2[A];
};

// One state, reference order. Returns the fp64 probability pair; logits out.
__device__ __forceinline__ void exact_forward(const ExactSmem& S, const float* __restrict__ xrow,
                                              double& p0, double& p1) {
    double x[F];
#pragma unroll
    for (int q = 0; q < F / 4; ++q) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(xrow) + q);
        x[4 * q] = v.x; x[4 * q + 1] = v.y; x[4 * q + 2] = v.z; x[4 * q + 3] = v.w;
    }
    double acc2[H2];
#pragma unroll
    for (int k = 0; k < H2; ++k) acc2[k] = S.b1[k];
#pragma unroll 1
    for (int j = 0; j < H1; ++j) {
        double z = S.b0[j];
        const double2* wr = reinterpret_cast<const double2*>(S.w0 + j * F);
#pragma unroll
        for (int q = 0; q < F / 2; ++q) {
            const double2 w = wr[q];
            // fp32*fp32 products are exact in fp64: fma == mul-then-add here
            z = fma(w.x, x[2 * q], z);
            z = fma(w.y, x[2 * q + 1], z);
        }
        const double h = z > 0.0 ? z : 0.0;
        const double2* w1c = reinterpret_cast<const double2*>(S.w1t + j * H2);
#pragma unroll
        for (int q = 0; q < H2 / 2; ++q) {
            const double2 w = w1c[q];
            acc2[2 * q] = madd_rn(acc2[2 * q], w.x, h);
            acc2[2 * q + 1] = madd_rn(acc2[2 * q + 1], w.y, h);
        }
    }
    double l0 = S.b2[0], l1 = S.b2[1];
#pragma unroll
    for (int k = 0; k < H2; ++k) {
        const double h = acc2[k] > 0.0 ? acc2[k] : 0.0;
        l0 = madd_rn(l0, S.w2[k], h);
        l1 = madd_rn(l1, S.w2[H2 + k], h);
    }
    const double m = fmax(l0, l1);
    const double e0 = exp(__dsub_rn(l0, m));
    const double e1 = exp(__dsub_rn(l1, m));
    const double s = __dadd_rn(e0, e1);
    p0 = __ddiv_rn(e0, s);
    p1 = __ddiv_rn(e1, s);
}

__device__ __forceinline__ void put_exact(ExactSmem& S, int t, float v) {
    if (t < OFF_B0) S.w0[t] = v;
    else if (t < OFF_W1) S.b0[t - OFF_B0] = v;
    else if (t < OFF_B1) {
        const int k = (t - OFF_W1) / H1, j = (t - OFF_W1) % H1;
        S.w1t[j * H2 + k] = v;
    } else if (t < OFF_W2) S.b1[t - OFF_B1] = v;
    else if (t < OFF_B2) S.w2[t - OFF_W2] = v;
    else S.b2[t - OFF_B2] = v;
}

// 16-byte loads, all of a thread's in flight at once (one memory round trip;
// the exact kernel keeps its 40 KB footprint for occupancy).
__device__ void load_exact_weights(ExactSmem& S, const float* __restrict__ p) {
    if ((reinterpret_cast<uintptr_t>(p) & 15u) == 0) {
        constexpr int NV = NP / 4, PER = (NV + EXACT_BLOCK - 1) / EXACT_BLOCK, CH = 4;
        // chunks of CH loads in flight: few registers (the kernel's occupancy
        // is set by its register count), ceil(PER / CH) round trips
#pragma unroll 1
        for (int u0 = 0; u0 < PER; u0 += CH) {
            float4 v[CH];
#pragma unroll
            for (int u = 0; u < CH; ++u) {
                const int c = threadIdx.x + (u0 + u) * EXACT_BLOCK;
                if (c < NV) v[u] = __ldg(reinterpret_cast<const float4*>(p) + c);
            }
#pragma unroll
            for (int u = 0; u < CH; ++u) {
                const int c = threadIdx.x + (u0 + u) * EXACT_BLOCK;
                if (c < NV) {
                    put_exact(S, 4 * c, v[u].x);
                    put_exact(S, 4 * c + 1, v[u].y);
                    put_exact(S, 4 * c + 2, v[u].z);
                    put_exact(S, 4 * c + 3, v[u].w);
                }
            }
        }
        for (int t = NV * 4 + threadIdx.x; t < NP; t += blockDim.x) put_exact(S, t, __ldg(p + t));
    } else {
        for (int t = threadIdx.x; t < NP; t += blockDim.x) put_exact(S, t, __ldg(p + t));
    }
    __syncthreads();
}

// Action + outputs of one exactly evaluated state (greedy or collection draw).
__device__ __forceinline__ void exact_finish(size_t s, double p0, double p1,
                                             double* __restrict__ probs, uint8_t* __restrict__ actions,
                                             const uint64_t* __restrict__ seg_off, size_t nseg,
                                             const uint64_t* __restrict__ seg_seed, double eps,
                                             int mode) {
    uint8_t act;
    if (mode & 8) {
        act = unit_of(sm_draw(seg_seed[0], (uint64_t)s + 1)) < p0 ? 0 : 1;
    } else if (mode & 4) {
        size_t lo = 0, hi = nseg;
        while (hi - lo > 1) {
            const size_t mid = (lo + hi) >> 1;
            if (seg_off[mid] <= s) lo = mid; else hi = mid;
        }
        const uint64_t j = s - seg_off[lo];
        const uint64_t seed = seg_seed[lo];
        const double ue = unit_of(sm_draw(seed, 2 * j + 1));
        const double ua = unit_of(sm_draw(seed, 2 * j + 2));
        act = ue < eps ? (ua < 0.5 ? 0 : 1) : (ua < p0 ? 0 : 1);
    } else {
        act = p1 >= p0 ? 1 : 0;  // ties -> Wave64 (policy.cpp:339-342)
    }
    if (mode & 2) actions[s] = act;
    if (mode & 1) {
        probs[2 * s] = p0;
        probs[2 * s + 1] = p1;
    }
}

// list == nullptr: all n states; else the n_list states named by list.
__global__ void __launch_bounds__(EXACT_BLOCK)
fwd_exact_kernel(const float* __restrict__ params, const float* __restrict__ feat, size_t n,
                 const uint32_t* __restrict__ list, const unsigned int* __restrict__ n_list,
                 double* __restrict__ probs, uint8_t* __restrict__ actions,
                 const uint64_t* __restrict__ seg_off, size_t nseg,
                 const uint64_t* __restrict__ seg_seed, double eps,
                 unsigned int* __restrict__ flags, int mode) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ExactSmem& S = *reinterpret_cast<ExactSmem*>(smem_raw);
    load_exact_weights(S, params);
    const size_t count = list ? (size_t)*n_list : n;
    for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < count;
         t += (size_t)gridDim.x * blockDim.x) {
        const size_t s = list ? (size_t)list[t] : t;
        const float* xrow = feat + s * F;
        if (!list) {
            bool finite = true;
            for (int i = 0; i < F; ++i) finite &= isfinite(xrow[i]);
            if (!finite) {
                atomicOr(flags, 1u);
                continue;
            }
        }
        double p0, p1;
        exact_forward(S, xrow, p0, p1);
        exact_finish(s, p0, p1, probs, actions, seg_off, nseg, seg_seed, eps, mode);
    }
}

// Re-check of the fast path's ambiguous states: one WARP per group of RS
// states (RS independent chains per lane hide the fp64 and shared-memory
// latencies; each weight read feeds RS states), so the short list finishes in
// a few group-latencies instead of one thread's full serial forward. Per
// output the operations and their order are exact_forward's (lane j: z_j over
// i ascending; lane k: acc2_k over j ascending; lane 2s+a: logit a of state s
// over k ascending), so the results are bit-identical.
constexpr int RS = 4;
struct RecheckScratch {
    double xs[RECHECK_BLOCK / 32][RS][F];
    double h1[RECHECK_BLOCK / 32][RS][H1];
    double h2[RECHECK_BLOCK / 32][RS][H2];
};
struct RecheckSmem {
    double w0t[F * H1];  // [i][j]: lane j reads consecutive words
    double w1t[H1 * H2]; // [j][k]
    double w2[A * H2];   // [a][k]
    double b0[H1];
    double b1[H2];
    double b2[A];
    union {  // the staged parameters are dead once the fp64 copies exist
        __align__(16) float raw[NP + 2];
        RecheckScratch sc;
    };
};

__global__ void __launch_bounds__(RECHECK_BLOCK)
fwd_recheck_kernel(const float* __restrict__ params, const float* __restrict__ feat,
                   const uint32_t* __restrict__ list, const unsigned int* __restrict__ n_list,
                   double* __restrict__ probs, uint8_t* __restrict__ actions,
                   const uint64_t* __restrict__ seg_off, size_t nseg,
                   const uint64_t* __restrict__ seg_seed, double eps, int mode) {
    constexpr int WPB = RECHECK_BLOCK / 32;
    const size_t count = *n_list;
    if ((size_t)blockIdx.x * WPB * RS >= count) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    RecheckSmem& S = *reinterpret_cast<RecheckSmem*>(smem_raw);
    stage_params(S.raw, params);
    for (int t = threadIdx.x; t < H1 * F; t += blockDim.x) {
        const int j = t / F, i = t - j * F;
        S.w0t[i * H1 + j] = S.raw[OFF_W0 + t];
    }
    for (int t = threadIdx.x; t < H1 * H2; t += blockDim.x) {
        const int k = t / H1, j = t % H1;
        S.w1t[j * H2 + k] = S.raw[OFF_W1 + t];
    }
    for (int t = threadIdx.x; t < A * H2; t += blockDim.x) S.w2[t] = S.raw[OFF_W2 + t];
    for (int t = threadIdx.x; t < H1; t += blockDim.x) S.b0[t] = S.raw[OFF_B0 + t];
    for (int t = threadIdx.x; t < H2; t += blockDim.x) S.b1[t] = S.raw[OFF_B1 + t];
    if (threadIdx.x < A) S.b2[threadIdx.x] = S.raw[OFF_B2 + threadIdx.x];
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (size_t g = ((size_t)blockIdx.x * WPB + w) * RS; g < count;
         g += (size_t)gridDim.x * WPB * RS) {
        const int nv = (int)min((size_t)RS, count - g);
        size_t sid[RS];
#pragma unroll
        for (int r = 0; r < RS; ++r) sid[r] = r < nv ? (size_t)list[g + r] : 0;
#pragma unroll
        for (int r = 0; r < RS; ++r) {
            const float* xrow = feat + sid[r] * F;
            S.sc.xs[w][r][lane] = r < nv ? (double)__ldg(xrow + lane) : 0.0;
            if (lane + 32 < F) S.sc.xs[w][r][lane + 32] = r < nv ? (double)__ldg(xrow + lane + 32) : 0.0;
        }
        __syncwarp();
        double za[RS], zb[RS];
#pragma unroll
        for (int r = 0; r < RS; ++r) { za[r] = S.b0[lane]; zb[r] = S.b0[lane + 32]; }
#pragma unroll 4
        for (int i = 0; i < F; ++i) {
            const double wa = S.w0t[i * H1 + lane], wb = S.w0t[i * H1 + lane + 32];
#pragma unroll
            for (int r = 0; r < RS; ++r) {
                const double x = S.sc.xs[w][r][i];
                za[r] = fma(wa, x, za[r]);  // exact products: fma == mul-then-add
                zb[r] = fma(wb, x, zb[r]);
            }
        }
#pragma unroll
        for (int r = 0; r < RS; ++r) {
            S.sc.h1[w][r][lane] = za[r] > 0.0 ? za[r] : 0.0;
            S.sc.h1[w][r][lane + 32] = zb[r] > 0.0 ? zb[r] : 0.0;
        }
        __syncwarp();
        double acc[RS];
#pragma unroll
        for (int r = 0; r < RS; ++r) acc[r] = S.b1[lane];
#pragma unroll 4
        for (int j = 0; j < H1; ++j) {
            const double wv = S.w1t[j * H2 + lane];
#pragma unroll
            for (int r = 0; r < RS; ++r) acc[r] = madd_rn(acc[r], wv, S.sc.h1[w][r][j]);
        }
#pragma unroll
        for (int r = 0; r < RS; ++r) S.sc.h2[w][r][lane] = acc[r] > 0.0 ? acc[r] : 0.0;
        __syncwarp();
        // lane 2r + a: logit a of state r
        const int lr = min(lane >> 1, RS - 1), la = lane & 1;
        double l = S.b2[la];
#pragma unroll 8
        for (int k = 0; k < H2; ++k) l = madd_rn(l, S.w2[la * H2 + k], S.sc.h2[w][lr][k]);
        const double l1 = __shfl_down_sync(0xffffffffu, l, 1);
        if (la == 0 && (lane >> 1) < nv) {
            const double l0 = l;
            const double m = fmax(l0, l1);
            const double e0 = exp(__dsub_rn(l0, m));
            const double e1 = exp(__dsub_rn(l1, m));
            const double sum = __dadd_rn(e0, e1);
            exact_finish((size_t)list[g + (lane >> 1)], __ddiv_rn(e0, sum),
                         __ddiv_rn(e1, sum), probs, actions, seg_off, nseg, seg_seed, eps, mode);
        }
        __syncwarp();  // scratch reuse
    }
}

size_t fast_smem_bytes() { return sizeof(FastSmem); }
size_t exact_smem_bytes() { return sizeof(ExactSmem); }
size_t recheck_smem_bytes() { return sizeof(RecheckSmem); }

}  // namespace gbxcu
