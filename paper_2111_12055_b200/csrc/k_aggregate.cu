// k_aggregate.cu — per-application reward aggregation (K3) for sm_100a.
//
// Replaces SimSuite::frame_time / run_benchmark (proj/src/simenv.cpp:439-510),
// the reward ratio of attribute_rewards / reward_from_framerate
// (proj/src/tuner.cpp:131-147, proj/src/core.cpp:125-133), and evaluate's
// uplift and 1%-bin histogram (proj/src/tuner.cpp:282-313).
//
// One warp per application (segment). The reference's per-app sums are strict
// left folds in pipeline -> slot order, so each warp loads 32 slots at a time
// (coalesced slot arrays, gathered shader latents/actions), forms the 32
// per-slot terms in parallel, and folds them in slot order with register
// shuffles — the serial part is one DADD per slot, everything else (gathers,
// products, divisions) is lane-parallel, and the loads run two chunks ahead
// of the fold (see SlotRaw). Results are bit-identical to the reference.
#include "common.cuh"
#include "kernels.h"

namespace gbxcu {

// acc (+|-)= term of lanes 0..count-1, in lane order. A full chunk is
// unrolled so every shuffle issues ahead of the serial DADD chain.
__device__ __forceinline__ double warp_fold(double acc, double term, int count, bool sub) {
    if (count == 32) {
#pragma unroll
        for (int k0 = 0; k0 < 32; k0 += 8) {
            double t[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) t[k] = __shfl_sync(0xffffffffu, term, k0 + k);
#pragma unroll
            for (int k = 0; k < 8; ++k) acc = sub ? __dsub_rn(acc, t[k]) : __dadd_rn(acc, t[k]);
        }
        return acc;
    }
    for (int k = 0; k < count; ++k) {
        const double t = __shfl_sync(0xffffffffu, term, k);
        acc = sub ? __dsub_rn(acc, t) : __dadd_rn(acc, t);
    }
    return acc;
}

// Slot stream of a warp: 32 slots per chunk, loads software-pipelined two
// chunks deep so the memory round trips overlap the (serial) fold of the
// current chunk: at chunk c the slot arrays of chunk c+2 and the gathers of
// chunk c+1 are in flight.
struct SlotRaw {
    uint32_t sh;
    double frac;
};

__device__ __forceinline__ SlotRaw slot_raw(const AggArgs& a, uint64_t s, uint64_t s_hi) {
    SlotRaw r{0xFFFFFFFFu, 0.0};
    if (s < s_hi) {
        r.sh = a.slot_shader[s];
        r.frac = a.slot_frac[s];
    }
    return r;
}

// pass-1 term of a slot: p * demand(a)
struct Term1In {
    double frac, bw;
    uint8_t act;
    bool ok;
};
__device__ __forceinline__ Term1In term1_gather(const AggArgs& a, const SlotRaw& r) {
    Term1In t{r.frac, 0.0, 0, r.sh != 0xFFFFFFFFu};
    if (t.ok) {
        t.bw = a.shader_lat[3 * (size_t)r.sh + 1];
        t.act = a.shader_action[r.sh];
    }
    return t;
}
__device__ __forceinline__ double term1(const Term1In& t) {
    if (!t.ok) return 0.0;
    const double demand = t.act == 1 ? __dmul_rn(2.0, t.bw) : t.bw;
    return __dmul_rn(t.frac, demand);
}

// pass-2 term of a slot: p / s_eff
struct Term2In {
    double frac, d, bw, kap;
    uint8_t act;
    bool ok;
};
__device__ __forceinline__ Term2In term2_gather(const AggArgs& a, const SlotRaw& r) {
    Term2In t{r.frac, 0.0, 0.0, 0.0, 0, r.sh != 0xFFFFFFFFu};
    if (t.ok) {
        const double* lat = a.shader_lat + 3 * (size_t)r.sh;
        t.d = lat[0];
        t.bw = lat[1];
        t.kap = lat[2];
        t.act = a.shader_action[r.sh];
    }
    return t;
}
__device__ __forceinline__ double term2(const Term2In& t, double thr, double throttle) {
    if (!t.ok) return 0.0;
    // wave64_speedup = (1 + kappa)(1 - 0.5 d)  (simenv.hpp:65-67)
    double sp = t.act == 1 ? __dmul_rn(__dadd_rn(1.0, t.kap), __dsub_rn(1.0, __dmul_rn(0.5, t.d))) : 1.0;
    if (t.bw > thr) sp = __dmul_rn(sp, throttle);
    return __ddiv_rn(t.frac, sp);
}

__global__ void __launch_bounds__(AGG_BLOCK) aggregate_kernel(AggArgs a) {
    const int lane = threadIdx.x & 31;
    const size_t warps = (size_t)gridDim.x * (AGG_BLOCK / 32);
    for (size_t app = (size_t)blockIdx.x * (AGG_BLOCK / 32) + (threadIdx.x >> 5); app < a.n_apps;
         app += warps) {
        const double baseline = a.app_f64[4 * app], cap = a.app_f64[4 * app + 1];
        const double sigma = a.app_f64[4 * app + 2], thr = a.app_f64[4 * app + 3];
        const uint64_t p_lo = a.app_pipe_off[app], p_hi = a.app_pipe_off[app + 1];

        // pass 1: bandwidth load = sum over all slots of p * demand(a) — the
        // app's slots are contiguous (pipelines in order), one stream
        double load = 0.0;
        {
            const uint64_t s_lo = a.pipe_slot_off[p_lo], s_hi = a.pipe_slot_off[p_hi];
            SlotRaw raw2 = slot_raw(a, s_lo + 32 + lane, s_hi);
            Term1In in1 = term1_gather(a, slot_raw(a, s_lo + lane, s_hi));
            for (uint64_t s0 = s_lo; s0 < s_hi; s0 += 32) {
                const double term = term1(in1);
                in1 = term1_gather(a, raw2);               // chunk c+1's gathers
                raw2 = slot_raw(a, s0 + 64 + lane, s_hi);  // chunk c+2's slot arrays
                load = warp_fold(load, term, (int)min((uint64_t)32, s_hi - s0), false);
            }
        }
        double throttle = 1.0;
        if (isfinite(cap) && load > cap) throttle = __ddiv_rn(cap, load);

        // pass 2: per pipeline inner = 1 - sum p + sum p / s_eff
        double total = 0.0;
        for (uint64_t p = p_lo; p < p_hi; ++p) {
            const uint64_t s_lo = a.pipe_slot_off[p], s_hi = a.pipe_slot_off[p + 1];
            double inner = 1.0;
            {
                double fnext = s_lo + lane < s_hi ? a.slot_frac[s_lo + lane] : 0.0;
                for (uint64_t s0 = s_lo; s0 < s_hi; s0 += 32) {
                    const double term = fnext;
                    fnext = s0 + 32 + lane < s_hi ? a.slot_frac[s0 + 32 + lane] : 0.0;
                    inner = warp_fold(inner, term, (int)min((uint64_t)32, s_hi - s0), true);
                }
            }
            {
                SlotRaw raw2 = slot_raw(a, s_lo + 32 + lane, s_hi);
                Term2In in2 = term2_gather(a, slot_raw(a, s_lo + lane, s_hi));
                for (uint64_t s0 = s_lo; s0 < s_hi; s0 += 32) {
                    const double term = term2(in2, thr, throttle);
                    in2 = term2_gather(a, raw2);
                    raw2 = slot_raw(a, s0 + 64 + lane, s_hi);
                    inner = warp_fold(inner, term, (int)min((uint64_t)32, s_hi - s0), false);
                }
            }
            const double wt = __dmul_rn(a.pipe_wt[2 * p], a.pipe_wt[2 * p + 1]);
            total = __dadd_rn(total, __dmul_rn(wt, inner));
        }
        const double fps = __ddiv_rn(1.0, total);

        // noisy samples: SplitMix64(derive_seed({run_seed, 0x4E5A45, app}))
        const uint64_t gapp = a.app_base + app;  // global app index (shards)
        const uint64_t run_seed =
            a.run_seed ? a.run_seed[app] : derive_seed3(a.eval_seed, 0x45564Cu, gapp);
        const uint64_t ns = derive_seed3(run_seed, 0x4E5A45u, gapp);
        const double half = __dmul_rn(sigma, sqrt(3.0));
        double sum = 0.0;
        for (int k0 = 0; k0 < a.n_samples; k0 += 32) {
            const int k = k0 + lane;
            double smp = 0.0;
            if (k < a.n_samples) {
                const double su = signed_unit_of(sm_draw(ns, (uint64_t)k + 1));
                smp = __dmul_rn(fps, __dadd_rn(1.0, __dmul_rn(su, half)));
                if (a.samples) a.samples[app * (size_t)a.n_samples + k] = smp;
            }
            sum = warp_fold(sum, smp, min(32, a.n_samples - k0), false);
        }
        if (lane == 0) {
            const double tuned = __ddiv_rn(sum, (double)a.n_samples);
            const double ratio = __ddiv_rn(tuned, baseline);
            double* row = a.rows + 5 * app;
            row[0] = total;
            row[1] = fps;
            row[2] = tuned;
            row[3] = __dmul_rn(100.0, __dsub_rn(ratio, 1.0));
            row[4] = ratio;
        }
    }
}

// evaluate's histogram (proj/src/tuner.cpp:293-313), one CTA.
__global__ void __launch_bounds__(1024)
histogram_kernel(const double* __restrict__ rows, int stride, size_t n, double* __restrict__ lower,
                 unsigned long long* __restrict__ count, size_t cap,
                 unsigned long long* __restrict__ n_bins) {
    __shared__ double s_lo[32], s_hi[32];
    __shared__ double s_lower;
    __shared__ unsigned long long s_bins;
    if (n == 0) {
        if (threadIdx.x == 0) *n_bins = 0;
        return;
    }
    double lo = rows[3], hi = rows[3];
    for (size_t k = threadIdx.x; k < n; k += blockDim.x) {
        const double u = rows[k * stride + 3];
        lo = fmin(lo, u);
        hi = fmax(hi, u);
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) { s_lo[w] = lo; s_hi[w] = hi; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i) { lo = fmin(lo, s_lo[i]); hi = fmax(hi, s_hi[i]); }
        const double lw = floor(lo);
        const double ch = ceil(hi);
        const double span = fmax(1.0, __dadd_rn(__dsub_rn(ch, lw), hi == ch ? 1.0 : 0.0));
        s_lower = lw;
        s_bins = (unsigned long long)span;
        *n_bins = s_bins;
    }
    __syncthreads();
    const double lw = s_lower;
    const unsigned long long bins = s_bins;
    for (size_t b = threadIdx.x; b < bins && b < cap; b += blockDim.x) {
        lower[b] = __dadd_rn(lw, (double)b);
        count[b] = 0;
    }
    __syncthreads();
    for (size_t k = threadIdx.x; k < n; k += blockDim.x) {
        unsigned long long idx = __double2ull_rz(__dsub_rn(rows[k * stride + 3], lw));
        if (idx > bins - 1) idx = bins - 1;
        if (idx < cap) atomicAdd(count + idx, 1ull);
    }
}

// [min, max] shader index referenced by slots [s_lo, s_hi) (an app-range
// shard infers only that shader range).
__global__ void slot_shader_range_kernel(const uint32_t* __restrict__ slot_shader, uint64_t s_lo,
                                         uint64_t s_hi, unsigned int* __restrict__ range) {
    unsigned int mn = 0xFFFFFFFFu, mx = 0u;
    for (uint64_t s = s_lo + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < s_hi;
         s += (uint64_t)gridDim.x * blockDim.x) {
        const unsigned int v = slot_shader[s];
        mn = min(mn, v);
        mx = max(mx, v);
    }
    for (int o = 16; o > 0; o >>= 1) {
        mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(range, mn);
        atomicMax(range + 1, mx);
    }
}

}  // namespace gbxcu
