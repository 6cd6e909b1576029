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
    float stats[8];     // R0,B0,R1,B1,R2,B2
};
static_assert(offsetof(FastSmem, w0) % 16 == 0 && offsetof(FastSmem, w1t) % 16 == 0, "align");

// Per-net constants of the guard: R_l = max_row ||w_row||_1, B_l = max |b|.
// Computed in fp64 and rounded up so the fp32 bound stays an upper bound.
__device__ void load_fast_weights(FastSmem& S, const float* __restrict__ p) {
    for (int t = threadIdx.x; t < H1 * F; t += blockDim.x) {
        const int j = t / F, i = t - j * F;  // coalesced read of w0[j][i]
        S.w0[(j >> 1) * (2 * F) + 2 * i + (j & 1)] = p[OFF_W0 + t];
    }
    for (int t = threadIdx.x; t < H1 * H2; t += blockDim.x) {
        const int k = t / H1, j = t % H1;  // coalesced read of w1[k][j]
        S.w1t[j * H2 + k] = p[OFF_W1 + t];
    }
    for (int t = threadIdx.x; t < A * H2; t += blockDim.x) S.w2[(t % H2) * A + t / H2] = p[OFF_W2 + t];
    for (int t = threadIdx.x; t < H1; t += blockDim.x) S.b0[t] = p[OFF_B0 + t];
    for (int t = threadIdx.x; t < H2; t += blockDim.x) S.b1[t] = p[OFF_B1 + t];
    if (threadIdx.x < A) S.b2[threadIdx.x] = p[OFF_B2 + threadIdx.x];
    __syncthreads();
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        double r0 = 0, bb0 = 0, r1 = 0, bb1 = 0, r2 = 0, bb2 = 0;
        for (int j = lane; j < H1; j += 32) {
            double s = 0;
            for (int i = 0; i < F; ++i) s += fabs((double)S.w0[(j >> 1) * (2 * F) + 2 * i + (j & 1)]);
            r0 = fmax(r0, s);
            bb0 = fmax(bb0, fabs((double)S.b0[j]));
        }
        {
            double s = 0;
            for (int j = 0; j < H1; ++j) s += fabs((double)S.w1t[j * H2 + lane]);
            r1 = s;
            bb1 = fabs((double)S.b1[lane]);
        }
        if (lane < A) {
            double s = 0;
            for (int k = 0; k < H2; ++k) s += fabs((double)S.w2[k * A + lane]);
            r2 = s;
            bb2 = fabs((double)S.b2[lane]);
        }
        for (int o = 16; o > 0; o >>= 1) {
            r0 = fmax(r0, __shfl_xor_sync(0xffffffffu, r0, o));
            bb0 = fmax(bb0, __shfl_xor_sync(0xffffffffu, bb0, o));
            r1 = fmax(r1, __shfl_xor_sync(0xffffffffu, r1, o));
            bb1 = fmax(bb1, __shfl_xor_sync(0xffffffffu, bb1, o));
            r2 = fmax(r2, __shfl_xor_sync(0xffffffffu, r2, o));
            bb2 = fmax(bb2, __shfl_xor_sync(0xffffffffu, bb2, o));
        }
        if (lane == 0) {
            // 1.0001 absorbs the rounding of the fp64 row sums themselves
            S.stats[0] = __double2float_ru(r0 * 1.0001);
            S.stats[1] = __double2float_ru(bb0);
            S.stats[2] = __double2float_ru(r1 * 1.0001);
            S.stats[3] = __double2float_ru(bb1);
            S.stats[4] = __double2float_ru(r2 * 1.0001);
            S.stats[5] = __double2float_ru(bb2);
        }
    }
    __syncthreads();
}

// Forward error bound on |(l1-l0)_fp32 - (l1-l0)_exact| (Higham-style
// recursive-summation bounds for FMA chains, u = 2^-24):
//   D1 = g(44)(B0 + R0 X)                      X  = max_i |x_i|
//   D2 = g(64)(B1 + R1 H1) + R1 D1             H1 = max_j h1_j  (fp32 values)
//   D3 = g(32)(B2 + R2 H2) + R2 D2             H2 = max_k h2_k
//   margin = 2 D3 (+1% slack; covers the fp64 reference's own rounding and
//   the rounding of this bound's evaluation), g(n) = (n+1) u (1 + 1e-4).
__device__ __forceinline__ float guard_threshold(const float* st, float X, float Hm1, float Hm2) {
    const float u = 5.9604645e-8f;  // 2^-24
    const float g44 = 45.f * u * 1.0001f, g64 = 65.f * u * 1.0001f, g32 = 33.f * u * 1.0001f;
    const float D1 = g44 * (st[1] + st[0] * X);
    const float D2 = g64 * (st[3] + st[2] * Hm1) + st[2] * D1;
    const float D3 = g32 * (st[5] + st[4] * Hm2) + st[4] * D2;
    return 2.02f * D3 + 1e-30f;
}

// Per-state tail of the fast path: guard, fp32 softmax, action (greedy or
// collection draw), re-check list, outputs.
__device__ __forceinline__ void fast_finish(const FastSmem& S, size_t s, float l0, float l1,
                                            float X, float hm1, float hm2, bool finite,
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
    const float T = guard_threshold(S.stats, X, hm1, hm2);
    const float d = l1 - l0;
    // fp32 softmax (max-subtracted like the reference)
    const float m = fmaxf(l0, l1);
    const float e0 = expf(l0 - m), e1 = expf(l1 - m);
    const float p0 = e0 / (e0 + e1);
    bool ambiguous;
    uint8_t act;
    if (mode & 4) {
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
__device__ __forceinline__ void fast_row(const float* xs, int r, float (&x)[F], float& X, bool& finite) {
    const float4* row = reinterpret_cast<const float4*>(xs + r * F);
#pragma unroll
    for (int q = 0; q < F / 4; ++q) {
        const float4 v = row[q];
        x[4 * q] = v.x; x[4 * q + 1] = v.y; x[4 * q + 2] = v.z; x[4 * q + 3] = v.w;
    }
    X = 0.f;
    finite = true;
#pragma unroll
    for (int i = 0; i < F; ++i) {
        finite &= isfinite(x[i]);
        X = fmaxf(X, fabsf(x[i]));
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
    load_fast_weights(S, params);

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
        float Xa, Xb;
        bool fa, fb;
        fast_row(xs, act0 ? lane : 0, xa, Xa, fa);
        fast_row(xs, act1 ? lane + 32 : 0, xb, Xb, fb);
        __syncwarp();  // the buffer is refilled two passes later

        // ---- layers 1+2 interleaved: acc2[k] += w1[k][j] * relu(z1_j), packed FFMA2
        float2 ca[H2 / 2], cb[H2 / 2];
#pragma unroll
        for (int q = 0; q < H2 / 2; ++q) ca[q] = cb[q] = make_float2(S.b1[2 * q], S.b1[2 * q + 1]);
        float hma = 0.f, hmb = 0.f;
#pragma unroll 2
        for (int jp = 0; jp < H1 / 2; ++jp) {
            const float4* wr = reinterpret_cast<const float4*>(S.w0 + jp * (2 * F));
            // two partial chains per z (even / odd inputs): twice the ILP; the
            // guard's error bound holds for any summation order
            float2 za = make_float2(S.b0[2 * jp], S.b0[2 * jp + 1]), zb = za;
            float2 za2 = make_float2(0.f, 0.f), zb2 = za2;
#pragma unroll
            for (int q = 0; q < F / 2; ++q) {
                const float4 w = wr[q];
                const float2 w01 = make_float2(w.x, w.y), w23 = make_float2(w.z, w.w);
                za = __ffma2_rn(w01, make_float2(xa[2 * q], xa[2 * q]), za);
                zb = __ffma2_rn(w01, make_float2(xb[2 * q], xb[2 * q]), zb);
                za2 = __ffma2_rn(w23, make_float2(xa[2 * q + 1], xa[2 * q + 1]), za2);
                zb2 = __ffma2_rn(w23, make_float2(xb[2 * q + 1], xb[2 * q + 1]), zb2);
            }
            za = make_float2(za.x + za2.x, za.y + za2.y);
            zb = make_float2(zb.x + zb2.x, zb.y + zb2.y);
            const float hA0 = za.x > 0.f ? za.x : 0.f, hA1 = za.y > 0.f ? za.y : 0.f;
            const float hB0 = zb.x > 0.f ? zb.x : 0.f, hB1 = zb.y > 0.f ? zb.y : 0.f;
            hma = fmaxf(hma, fmaxf(hA0, hA1));
            hmb = fmaxf(hmb, fmaxf(hB0, hB1));
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
            fast_finish(S, base + lane, la.x, la.y, Xa, hma, h2a, fa, probs, actions, seg_off, nseg,
                        seg_seed, eps, recheck, n_recheck, flags, mode);
        if (act1)
            fast_finish(S, base + 32 + lane, lb.x, lb.y, Xb, hmb, h2b, fb, probs, actions, seg_off,
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

__device__ void load_exact_weights(ExactSmem& S, const float* __restrict__ p) {
    for (int t = threadIdx.x; t < H1 * F; t += blockDim.x) S.w0[t] = p[OFF_W0 + t];
    for (int t = threadIdx.x; t < H1 * H2; t += blockDim.x) {
        const int k = t / H1, j = t % H1;
        S.w1t[j * H2 + k] = p[OFF_W1 + t];
    }
    for (int t = threadIdx.x; t < A * H2; t += blockDim.x) S.w2[t] = p[OFF_W2 + t];
    for (int t = threadIdx.x; t < H1; t += blockDim.x) S.b0[t] = p[OFF_B0 + t];
    for (int t = threadIdx.x; t < H2; t += blockDim.x) S.b1[t] = p[OFF_B1 + t];
    if (threadIdx.x < A) S.b2[threadIdx.x] = p[OFF_B2 + threadIdx.x];
    __syncthreads();
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
        uint8_t act;
        if (mode & 4) {
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
}

size_t fast_smem_bytes() { return sizeof(FastSmem); }
size_t exact_smem_bytes() { return sizeof(ExactSmem); }

}  // namespace gbxcu
