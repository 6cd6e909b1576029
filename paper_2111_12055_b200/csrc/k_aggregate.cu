// k_aggregate.cu — per-application reward aggregation (K3) for sm_100a.
//
// Replaces SimSuite::frame_time / run_benchmark (proj/src/simenv.cpp:439-510),
// the reward ratio of attribute_rewards / reward_from_framerate
// (proj/src/tuner.cpp:131-147, proj/src/core.cpp:125-133), and evaluate's
// uplift and 1%-bin histogram (proj/src/tuner.cpp:282-313).
//
// A warp folds AGG_APPS applications at once (lane j = app j) over terms the
// whole warp forms lane-parallel; see aggregate_kernel below. Results are
// bit-identical to the reference.
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

// ---------------------------------------------------------------- K3 kernel
// K applications per warp. The reference's sums are strict left folds,
// so an app's folds are serial; what a warp can share is the fold
// *instruction*: lane j (< K) folds app j while the whole warp loads
// and forms the per-slot terms of every app's next 32-slot chunk
// lane-parallel (coalesced slot arrays, gathered shader latents / actions)
// and stages them in shared memory. One fold instruction thus advances
// K apps by one slot; the warp-per-app form spent one DADD and one
// SHFL per slot and pass on a single app and was issue-bound (ncu: 58% issue
// active, MIO throttle the top stall).
//
// One streaming read per pipeline: run_benchmark's bandwidth load (pass 1,
// over all the app's slots) and each pipeline's inner sum (pass 2: 1 - sum p,
// then + sum p / s_eff) are folded in the reference's order, with the pass-2
// terms formed under the speculation that the app is not throttled
// (throttle == 1, so s_eff is the wave64 speedup exactly). Per pipeline that
// is an "A" segment (its fractions: inner -= p) then a "B" segment (load +=
// p * demand, inner += p / s_eff): 45 B read per slot instead of the 82 B of
// three separate passes (the A read is mostly an L2 hit for B). An app whose
// final load exceeds its cap (throttle != 1) runs pass 2 again with the true
// throttle ("redo" segments, which leave the load unchanged). Bit-identical to
// the reference either way.
struct AggLane {  // lanes < K: app `lane`'s fold cursor
    uint64_t pos, end;  // slots still to fold in the current segment
    uint64_t p, p_lo, p_hi;
    double load, inner, total, throttle, cap;
    int seg;   // 0 = A (fractions), 1 = B (terms), 2 = done
    int redo;  // pass 2 again with the app's true throttle
};

__device__ __forceinline__ void agg_start_pipeline(const AggArgs& a, AggLane& L) {
    L.seg = 0;
    L.inner = 1.0;
    L.pos = a.pipe_slot_off[L.p];
    L.end = a.pipe_slot_off[L.p + 1];
}

// past the end of the current segment: on to the next non-empty one (or done)
__device__ void agg_advance(const AggArgs& a, AggLane& L) {
    while (L.seg != 2 && L.pos >= L.end) {
        if (L.seg == 0) {  // A -> B over the same pipeline
            L.seg = 1;
            L.pos = a.pipe_slot_off[L.p];
            L.end = a.pipe_slot_off[L.p + 1];
            continue;
        }
        // B done: the pipeline's weighted inner sum (frame_time, simenv.cpp:439-474)
        const double wt = __dmul_rn(a.pipe_wt[2 * L.p], a.pipe_wt[2 * L.p + 1]);
        L.total = __dadd_rn(L.total, __dmul_rn(wt, L.inner));
        if (++L.p < L.p_hi) {
            agg_start_pipeline(a, L);
            continue;
        }
        if (!L.redo) {  // end of the app's load: its throttle
            double thr = 1.0;
            if (isfinite(L.cap) && L.load > L.cap) thr = __ddiv_rn(L.cap, L.load);
            L.throttle = thr;
            if (thr != 1.0) {
                L.redo = 1;
                L.total = 0.0;
                L.p = L.p_lo;
                agg_start_pipeline(a, L);
                continue;
            }
        }
        L.seg = 2;
    }
}

template <int K, int MINB>
__global__ void __launch_bounds__(AGG_BLOCK, MINB) aggregate_kernel(AggArgs a) {
    __shared__ double2 buf[AGG_BLOCK / 32][K][33];  // staged (load term, inner term)
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const size_t warps = (size_t)gridDim.x * (AGG_BLOCK / 32);
    const size_t n_groups = (a.n_apps + K - 1) / K;
    for (size_t grp = (size_t)blockIdx.x * (AGG_BLOCK / 32) + wib; grp < n_groups; grp += warps) {
        const size_t app0 = grp * K;
        AggLane L{};
        L.seg = 2;
        L.throttle = 1.0;
        double thr_me = 0.0;
        if (lane < K && app0 + lane < a.n_apps) {
            const size_t app = app0 + lane;
            L.cap = a.app_f64[4 * app + 1];
            thr_me = a.app_f64[4 * app + 3];
            L.p_lo = L.p = a.app_pipe_off[app];
            L.p_hi = a.app_pipe_off[app + 1];
            if (L.p < L.p_hi) {
                agg_start_pipeline(a, L);
                agg_advance(a, L);  // (empty leading segments)
            }
        }
        for (;;) {
            // this round's chunk of every app: (segment | redo | count), start, threshold, throttle
            const int cnt_me = L.seg == 2 ? 0 : (int)min((uint64_t)32, L.end - L.pos);
            const int info_me = cnt_me | (L.seg << 8) | (L.redo << 10);
            int info[K];
            uint64_t pos[K];
#pragma unroll
            for (int j = 0; j < K; ++j) {
                info[j] = __shfl_sync(0xffffffffu, info_me, j);
                pos[j] = __shfl_sync(0xffffffffu, L.pos, j);
            }
            bool any = false;
#pragma unroll
            for (int j = 0; j < K; ++j) any |= (info[j] & 0xFF) != 0;
            if (!any) break;
            // loads: slot arrays of every app's chunk, then the shader gathers
            double fr[K];
            uint32_t sh[K];
#pragma unroll
            for (int j = 0; j < K; ++j) {
                const bool ok = lane < (info[j] & 0xFF);
                fr[j] = ok ? a.slot_frac[pos[j] + lane] : 0.0;
                sh[j] = ok && (info[j] >> 8 & 3) == 1 ? a.slot_shader[pos[j] + lane] : 0xFFFFFFFFu;
            }
            double ld[K], lb[K], lk[K];
            uint8_t ac[K];
#pragma unroll
            for (int j = 0; j < K; ++j) {
                ld[j] = lb[j] = lk[j] = 0.0;
                ac[j] = 0;
                if (sh[j] != 0xFFFFFFFFu) {
                    const double* lat = a.shader_lat + 3 * (size_t)sh[j];
                    ld[j] = lat[0];
                    lb[j] = lat[1];
                    lk[j] = lat[2];
                    ac[j] = a.shader_action[sh[j]];
                }
            }
            // terms
#pragma unroll
            for (int j = 0; j < K; ++j) {
                const double thr = __shfl_sync(0xffffffffu, thr_me, j);
                const double throttle = __shfl_sync(0xffffffffu, L.throttle, j);
                // (-0.0 pads the chunk: x + (-0.0) == x for every x, so the
                //  folds below need no per-slot predicate)
                double x = -0.0, y = -0.0;
                if (lane < (info[j] & 0xFF)) {
                    x = 0.0;
                    if ((info[j] >> 8 & 3) == 0) {
                        y = -fr[j];  // inner - p == inner + (-p) exactly
                    } else {
                        // pass 1: p * demand(a) (simenv.cpp:481-510)
                        if (!(info[j] >> 10 & 1))
                            x = __dmul_rn(fr[j], ac[j] == 1 ? __dmul_rn(2.0, lb[j]) : lb[j]);
                        // pass 2: p / s_eff, wave64_speedup = (1 + kappa)(1 - 0.5 d)
                        double sp = ac[j] == 1 ? __dmul_rn(__dadd_rn(1.0, lk[j]),
                                                           __dsub_rn(1.0, __dmul_rn(0.5, ld[j])))
                                               : 1.0;
                        if (lb[j] > thr) sp = __dmul_rn(sp, throttle);
                        y = sp == 1.0 ? fr[j] : __ddiv_rn(fr[j], sp);  // (p / 1 == p exactly)
                    }
                }
                buf[wib][j][lane] = make_double2(x, y);
            }
            __syncwarp();
            // folds: lane j folds app j's chunk in slot order
            if (lane < K) {
#pragma unroll
                for (int k = 0; k < 32; ++k) {
                    const double2 t = buf[wib][lane][k];
                    L.load = __dadd_rn(L.load, t.x);
                    L.inner = __dadd_rn(L.inner, t.y);
                }
                L.pos += cnt_me;
                agg_advance(a, L);
            }
            __syncwarp();
        }

        // per app: noisy samples SplitMix64(derive_seed({run_seed, 0x4E5A45, app})),
        // tuned fps, uplift and reward ratio (tuner.cpp:276-291, core.cpp:125-133)
        for (int j = 0; j < K && app0 + j < a.n_apps; ++j) {
            const size_t app = app0 + j;
            const double total = __shfl_sync(0xffffffffu, L.total, j);
            const double fps = __ddiv_rn(1.0, total);
            const double baseline = a.app_f64[4 * app], sigma = a.app_f64[4 * app + 2];
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
}

// AGG_APPS apps per warp, 3 CTAs per SM (register cap 80): measured at C5
// (1e8 slots, 1e4 apps) against 1/2/8 apps per warp and 2-4 CTAs per SM
// (profiles/r02/k3_variants.md)
template __global__ void aggregate_kernel<AGG_APPS, AGG_MINB>(AggArgs);

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
