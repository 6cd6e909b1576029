// k_train.cu — fused minibatch train step (K1) for sm_100a, fp64 parity mode.
//
// Replaces fit's inner loop (proj/src/policy.cpp:316-333): batch_kl_loss,
// batch_kl_gradient (forward + analytic backward, :209-279) and the SGD
// update w = float(double(w) - lr * g) (:328-332).
//
// Every stage is a small dense contraction whose reduction (K) dimension is
// kept SEQUENTIAL inside one thread — exactly the reference's summation order
// — while M/N are spread over the CTA with register blocking:
//   F1 h1[r][j]  = relu(b0[j] + sum_i x[r][i]  w0[j][i])   K = 44  (DFMA: products exact)
//   F2 h2[r][k]  = relu(b1[k] + sum_j h1[r][j] w1[k][j])   K = 64  (mul, then add)
//   F3 logits, softmax, KL, d3 = p (ln(p^/t^) - L) / |b|
//   B1 d2[r][k]  = d3[r][0] w2[0][k] + d3[r][1] w2[1][k], masked by h2 > 0
//   B2 d1[r][j]  = sum_k d2[r][k] w1[k][j], masked by h1 > 0
//   G  gw2/gw1/gw0/gb* += per-record outer products, K = records in batch order
// Gradient accumulators are owned by threads (registers) across all tiles of a
// step, so a 1-CTA step reproduces the reference's per-parameter left fold bit
// for bit (up to exp/log ulps). Multi-CTA steps reduce per-CTA partials in
// CTA order (fp64; differs from the reference only in re-association).
//
// Modes
//   FUSED  : one launch = one epoch; G CTAs; in-kernel deterministic
//            cross-CTA reduction + SGD with a grid barrier (cooperative launch).
//   PARTIAL: one launch = one step's per-CTA partial gradients (data-parallel
//            path; reduction, NCCL all-reduce and update run in follow-up
//            kernels, see gbxcu_api.cu).
#include <cstddef>

#include "common.cuh"
#include "kernels.h"

namespace gbxcu {

struct TrainSmem {
    double w0t[F * H1];  // [i][j]
    double w1[H2 * H1];  // [k][j]
    double w1t[H1 * H2]; // [j][k]
    double w2[A * H2];   // [a][k]
    double b0[H1];
    double b1[H2];
    double b2[A];
    double x[TB * F];    // [r][i]
    double h1[TB * H1];  // [r][j]
    double h2[TB * H2];  // [r][k]
    double d2[TB * H2];  // [r][k]
    double d1[TB * H1];  // [r][j]
    double d3[TB * 2];
    double tgt[TB * 2];
    double kl[TB];
    double scal[4];      // [0] step loss total, [1] loss, [2] diverged flag
};

static_assert(offsetof(TrainSmem, x) % 16 == 0 && offsetof(TrainSmem, h1) % 16 == 0 &&
                  offsetof(TrainSmem, d2) % 16 == 0 && offsetof(TrainSmem, d1) % 16 == 0,
              "double2 loads need 16-byte alignment");

size_t train_smem_bytes() { return sizeof(TrainSmem); }

__device__ void load_train_weights(TrainSmem& S, const float* __restrict__ p) {
    for (int t = threadIdx.x; t < H1 * F; t += blockDim.x) {
        const int j = t / F, i = t % F;
        S.w0t[i * H1 + j] = p[OFF_W0 + t];
    }
    for (int t = threadIdx.x; t < H2 * H1; t += blockDim.x) {
        const double w = p[OFF_W1 + t];
        const int k = t / H1, j = t % H1;
        S.w1[t] = w;
        S.w1t[j * H2 + k] = w;
    }
    for (int t = threadIdx.x; t < A * H2; t += blockDim.x) S.w2[t] = p[OFF_W2 + t];
    for (int t = threadIdx.x; t < H1; t += blockDim.x) S.b0[t] = p[OFF_B0 + t];
    for (int t = threadIdx.x; t < H2; t += blockDim.x) S.b1[t] = p[OFF_B1 + t];
    if (threadIdx.x < A) S.b2[threadIdx.x] = p[OFF_B2 + threadIdx.x];
}

// Thread-owned gradient accumulators for one step.
struct GradRegs {
    double g0a[8], g0b[8];  // gw0[8w+jj][lane], gw0[8w+jj][lane+32] (lane < 12)
    double g1[4][2];        // gw1[4w+kk][lane + 32q]
    double gx;              // tid<64: gb0[tid]; <96: gb1; <160: gw2; <162: gb2
    double loss;            // tid 0: running sum of per-record KL (batch order)
};

__device__ __forceinline__ void zero_grads(GradRegs& g) {
#pragma unroll
    for (int q = 0; q < 8; ++q) g.g0a[q] = g.g0b[q] = 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) g.g1[q][0] = g.g1[q][1] = 0.0;
    g.gx = 0.0;
    g.loss = 0.0;
}

// Flat parameter index owned by slot (used for partial writes and updates).
// Visits every owned (flat index, accumulator) pair.
template <typename Fn>
__device__ __forceinline__ void for_each_owned(GradRegs& g, Fn fn) {
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
        const int j = 8 * w + jj;
        fn(OFF_W0 + j * F + lane, g.g0a[jj]);
        if (lane < F - 32) fn(OFF_W0 + j * F + lane + 32, g.g0b[jj]);
    }
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
#pragma unroll
        for (int q = 0; q < 2; ++q) fn(OFF_W1 + (4 * w + kk) * H1 + lane + 32 * q, g.g1[kk][q]);
    if (tid < 64) fn(OFF_B0 + tid, g.gx);
    else if (tid < 96) fn(OFF_B1 + tid - 64, g.gx);
    else if (tid < 160) fn(OFF_W2 + tid - 96, g.gx);
    else if (tid < 162) fn(OFF_B2 + tid - 160, g.gx);
}

// Write a new fp32 parameter value (as double) into every smem copy.
__device__ __forceinline__ void set_smem_param(TrainSmem& S, int p, double v) {
    if (p < OFF_B0) { const int j = p / F, i = p % F; S.w0t[i * H1 + j] = v; }
    else if (p < OFF_W1) S.b0[p - OFF_B0] = v;
    else if (p < OFF_B1) {
        const int t = p - OFF_W1, k = t / H1, j = t % H1;
        S.w1[t] = v;
        S.w1t[j * H2 + k] = v;
    } else if (p < OFF_W2) S.b1[p - OFF_B1] = v;
    else if (p < OFF_B2) S.w2[p - OFF_W2] = v;
    else S.b2[p - OFF_B2] = v;
}

__device__ __forceinline__ double get_smem_param(const TrainSmem& S, int p) {
    if (p < OFF_B0) { const int j = p / F, i = p % F; return S.w0t[i * H1 + j]; }
    if (p < OFF_W1) return S.b0[p - OFF_B0];
    if (p < OFF_B1) return S.w1[p - OFF_W1];
    if (p < OFF_W2) return S.b1[p - OFF_B1];
    if (p < OFF_B2) return S.w2[p - OFF_W2];
    return S.b2[p - OFF_B2];
}

// Process up to TB records rows[0..nv) of the batch; accumulates into g.
__device__ void train_tile(TrainSmem& S, GradRegs& g, const float* __restrict__ feat,
                           const double* __restrict__ tgt, const uint32_t* __restrict__ order,
                           size_t row0, int nv, double inv_b) {
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    // ---- P0: gather records (zero-fill rows past nv)
    for (int t = tid; t < TB * (F / 4); t += TRAIN_BLOCK) {
        const int r = t / (F / 4), q = t % (F / 4);
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (r < nv) {
            const size_t rec = order[row0 + r];
            v = __ldg(reinterpret_cast<const float4*>(feat + rec * F) + q);
        }
        double* xr = S.x + r * F + 4 * q;
        xr[0] = v.x; xr[1] = v.y; xr[2] = v.z; xr[3] = v.w;
    }
    if (tid < TB) {
        double t0 = 0.5, t1 = 0.5;
        if (tid < nv) {
            const size_t rec = order[row0 + tid];
            t0 = tgt[2 * rec];
            t1 = tgt[2 * rec + 1];
        }
        S.tgt[2 * tid] = t0;
        S.tgt[2 * tid + 1] = t1;
    }
    __syncthreads();

    // ---- F1: lanes <-> j (lane, lane+32), warp <-> rows 8w..8w+7
    {
        double acc[8][2];
        const double bA = S.b0[lane], bB = S.b0[lane + 32];
#pragma unroll
        for (int rr = 0; rr < 8; ++rr) { acc[rr][0] = bA; acc[rr][1] = bB; }
        const double* xb = S.x + (8 * w) * F;
#pragma unroll 2
        for (int i = 0; i < F; i += 2) {
            const double wA0 = S.w0t[i * H1 + lane], wB0 = S.w0t[i * H1 + lane + 32];
            const double wA1 = S.w0t[(i + 1) * H1 + lane], wB1 = S.w0t[(i + 1) * H1 + lane + 32];
#pragma unroll
            for (int rr = 0; rr < 8; ++rr) {
                const double2 xv = *reinterpret_cast<const double2*>(xb + rr * F + i);
                acc[rr][0] = fma(wA0, xv.x, acc[rr][0]);
                acc[rr][1] = fma(wB0, xv.x, acc[rr][1]);
                acc[rr][0] = fma(wA1, xv.y, acc[rr][0]);
                acc[rr][1] = fma(wB1, xv.y, acc[rr][1]);
            }
        }
#pragma unroll
        for (int rr = 0; rr < 8; ++rr) {
            double* hr = S.h1 + (8 * w + rr) * H1;
            hr[lane] = acc[rr][0] > 0.0 ? acc[rr][0] : 0.0;
            hr[lane + 32] = acc[rr][1] > 0.0 ? acc[rr][1] : 0.0;
        }
    }
    __syncthreads();

    // ---- F2: lanes <-> k, warp <-> rows
    {
        double acc[8];
        const double b = S.b1[lane];
#pragma unroll
        for (int rr = 0; rr < 8; ++rr) acc[rr] = b;
        const double* hb = S.h1 + (8 * w) * H1;
#pragma unroll 2
        for (int j = 0; j < H1; j += 2) {
            const double w0 = S.w1t[j * H2 + lane], w1 = S.w1t[(j + 1) * H2 + lane];
#pragma unroll
            for (int rr = 0; rr < 8; ++rr) {
                const double2 hv = *reinterpret_cast<const double2*>(hb + rr * H1 + j);
                acc[rr] = madd_rn(acc[rr], w0, hv.x);
                acc[rr] = madd_rn(acc[rr], w1, hv.y);
            }
        }
#pragma unroll
        for (int rr = 0; rr < 8; ++rr)
            S.h2[(8 * w + rr) * H2 + lane] = acc[rr] > 0.0 ? acc[rr] : 0.0;
    }
    __syncthreads();

    // ---- F3 + loss + d3: one thread per row
    if (tid < TB) {
        const int r = tid;
        double l0 = S.b2[0], l1 = S.b2[1];
        const double* h = S.h2 + r * H2;
#pragma unroll 8
        for (int k = 0; k < H2; ++k) {
            l0 = madd_rn(l0, S.w2[k], h[k]);
            l1 = madd_rn(l1, S.w2[H2 + k], h[k]);
        }
        const double m = fmax(l0, l1);
        const double e0 = exp(__dsub_rn(l0, m)), e1 = exp(__dsub_rn(l1, m));
        const double s = __dadd_rn(e0, e1);
        const double p[2] = {__ddiv_rn(e0, s), __ddiv_rn(e1, s)};
        double lr[2], loss = 0.0;
#pragma unroll
        for (int a = 0; a < 2; ++a) {
            const double pc = clampp(p[a]);
            const double tc = clampp(S.tgt[2 * r + a]);
            lr[a] = log(__ddiv_rn(pc, tc));
            loss = madd_rn(loss, pc, lr[a]);
        }
        const bool valid = r < nv;
        S.kl[r] = valid ? loss : 0.0;
#pragma unroll
        for (int a = 0; a < 2; ++a)
            S.d3[2 * r + a] = valid ? __dmul_rn(__dmul_rn(p[a], __dsub_rn(lr[a], loss)), inv_b) : 0.0;
    }
    __syncthreads();

    // ---- B1: d2 = (0 + d3_0 w2_0k) + d3_1 w2_1k, masked by h2 > 0
    {
        const double w20 = S.w2[lane], w21 = S.w2[H2 + lane];
#pragma unroll
        for (int rr = 0; rr < 8; ++rr) {
            const int r = 8 * w + rr;
            double d = madd_rn(0.0, S.d3[2 * r], w20);
            d = madd_rn(d, S.d3[2 * r + 1], w21);
            S.d2[r * H2 + lane] = S.h2[r * H2 + lane] <= 0.0 ? 0.0 : d;
        }
    }
    if (tid == 0) {
        for (int r = 0; r < nv; ++r) g.loss = __dadd_rn(g.loss, S.kl[r]);
    }
    __syncthreads();

    // ---- B2: d1[r][j] = sum_k d2[r][k] w1[k][j], masked by h1 > 0
    //      (+ gw1/gb1/gw2/gb2 accumulation, which only needs d2/d3/h1/h2)
    {
        double acc[8][2];
#pragma unroll
        for (int rr = 0; rr < 8; ++rr) acc[rr][0] = acc[rr][1] = 0.0;
        const double* db = S.d2 + (8 * w) * H2;
#pragma unroll 2
        for (int k = 0; k < H2; k += 2) {
            const double wA0 = S.w1[k * H1 + lane], wB0 = S.w1[k * H1 + lane + 32];
            const double wA1 = S.w1[(k + 1) * H1 + lane], wB1 = S.w1[(k + 1) * H1 + lane + 32];
#pragma unroll
            for (int rr = 0; rr < 8; ++rr) {
                const double2 dv = *reinterpret_cast<const double2*>(db + rr * H2 + k);
                // rows with d2 == 0 add a signed zero: a no-op, matching the
                // reference's `continue` (policy.cpp:247)
                acc[rr][0] = madd_rn(acc[rr][0], dv.x, wA0);
                acc[rr][1] = madd_rn(acc[rr][1], dv.x, wB0);
                acc[rr][0] = madd_rn(acc[rr][0], dv.y, wA1);
                acc[rr][1] = madd_rn(acc[rr][1], dv.y, wB1);
            }
        }
#pragma unroll
        for (int rr = 0; rr < 8; ++rr) {
            const int r = 8 * w + rr;
            S.d1[r * H1 + lane] = S.h1[r * H1 + lane] <= 0.0 ? 0.0 : acc[rr][0];
            S.d1[r * H1 + lane + 32] = S.h1[r * H1 + lane + 32] <= 0.0 ? 0.0 : acc[rr][1];
        }
        // gw1[4w+kk][lane+32q] += d2[r][4w+kk] * h1[r][lane+32q], r in batch order
        for (int r = 0; r < nv; ++r) {
            const double2 da = *reinterpret_cast<const double2*>(S.d2 + r * H2 + 4 * w);
            const double2 dbv = *reinterpret_cast<const double2*>(S.d2 + r * H2 + 4 * w + 2);
            const double hA = S.h1[r * H1 + lane], hB = S.h1[r * H1 + lane + 32];
            g.g1[0][0] = madd_rn(g.g1[0][0], da.x, hA);
            g.g1[0][1] = madd_rn(g.g1[0][1], da.x, hB);
            g.g1[1][0] = madd_rn(g.g1[1][0], da.y, hA);
            g.g1[1][1] = madd_rn(g.g1[1][1], da.y, hB);
            g.g1[2][0] = madd_rn(g.g1[2][0], dbv.x, hA);
            g.g1[2][1] = madd_rn(g.g1[2][1], dbv.x, hB);
            g.g1[3][0] = madd_rn(g.g1[3][0], dbv.y, hA);
            g.g1[3][1] = madd_rn(g.g1[3][1], dbv.y, hB);
        }
        if (tid >= 64 && tid < 96) {
            const int k = tid - 64;
            for (int r = 0; r < nv; ++r) g.gx = __dadd_rn(g.gx, S.d2[r * H2 + k]);
        } else if (tid >= 96 && tid < 160) {
            const int a = (tid - 96) / H2, k = (tid - 96) % H2;
            for (int r = 0; r < nv; ++r) g.gx = madd_rn(g.gx, S.d3[2 * r + a], S.h2[r * H2 + k]);
        } else if (tid >= 160 && tid < 162) {
            const int a = tid - 160;
            for (int r = 0; r < nv; ++r) g.gx = __dadd_rn(g.gx, S.d3[2 * r + a]);
        }
    }
    __syncthreads();

    // ---- G0: gw0[8w+jj][i] += d1[r][8w+jj] * x[r][i]; gb0[j] += d1[r][j]
    {
        const bool two = lane < F - 32;
        for (int r = 0; r < nv; ++r) {
            const double* dr = S.d1 + r * H1 + 8 * w;
            const double2 d01 = *reinterpret_cast<const double2*>(dr);
            const double2 d23 = *reinterpret_cast<const double2*>(dr + 2);
            const double2 d45 = *reinterpret_cast<const double2*>(dr + 4);
            const double2 d67 = *reinterpret_cast<const double2*>(dr + 6);
            const double dv[8] = {d01.x, d01.y, d23.x, d23.y, d45.x, d45.y, d67.x, d67.y};
            const double xa = S.x[r * F + lane];
            const double xb = two ? S.x[r * F + lane + 32] : 0.0;
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
                g.g0a[jj] = madd_rn(g.g0a[jj], dv[jj], xa);
                g.g0b[jj] = madd_rn(g.g0b[jj], dv[jj], xb);
            }
        }
        if (tid < 64) {
            for (int r = 0; r < nv; ++r) g.gx = __dadd_rn(g.gx, S.d1[r * H1 + tid]);
        }
    }
    __syncthreads();
}

// Records of step `step` handled by CTA `cta` of `nctas` on rank `rank` of
// `nranks`: equal contiguous slices of the global batch, rank-major.
__device__ __forceinline__ void step_slice(size_t n, int batch, long step, int rank, int nranks,
                                           int cta, int nctas, size_t& lo, size_t& hi,
                                           size_t& nb) {
    const size_t start = (size_t)step * (size_t)batch;
    const size_t stop = min(n, start + (size_t)batch);
    nb = stop - start;
    const size_t per_rank = (nb + nranks - 1) / nranks;
    const size_t r_lo = min(stop, start + (size_t)rank * per_rank);
    const size_t r_hi = min(stop, r_lo + per_rank);
    const size_t m = r_hi - r_lo;
    const size_t per_cta = (m + nctas - 1) / nctas;
    lo = min(r_hi, r_lo + (size_t)cta * per_cta);
    hi = min(r_hi, lo + per_cta);
}

__device__ void run_step_tiles(TrainSmem& S, GradRegs& g, const TrainArgs& a, long step,
                               size_t& nb) {
    size_t lo, hi;
    step_slice(a.n, a.batch, step, a.rank, a.nranks, blockIdx.x, gridDim.x, lo, hi, nb);
    const double inv_b = 1.0 / (double)nb;  // batch_kl_gradient's 1/|b| (global batch)
    for (size_t r0 = lo; r0 < hi; r0 += TB) {
        const int nv = (int)min((size_t)TB, hi - r0);
        train_tile(S, g, a.feat, a.tgt, a.order, r0, nv, inv_b);
    }
}

__global__ void __launch_bounds__(TRAIN_BLOCK, 1) train_epoch_kernel(TrainArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TrainSmem& S = *reinterpret_cast<TrainSmem*>(smem_raw);
    if (*a.diverged_epoch >= 0) return;  // an earlier epoch diverged
    load_train_weights(S, a.params);
    __syncthreads();
    GradRegs g;
    zero_grads(g);
    unsigned int bar_target = 0;
    const bool single = gridDim.x == 1;
    double epoch_total = 0.0;
    const long n_steps = (long)((a.n + a.batch - 1) / a.batch);

    for (long step = 0; step < n_steps; ++step) {
        size_t nb;
        run_step_tiles(S, g, a, step, nb);
        if (single) {
            // loss = (sum of per-record KL, batch order) / |b|  (policy.cpp:194-201)
            if (threadIdx.x == 0) {
                const double loss = __ddiv_rn(g.loss, (double)nb);
                S.scal[1] = loss;
                S.scal[2] = isfinite(loss) ? 0.0 : 1.0;
            }
            __syncthreads();
            if (S.scal[2] != 0.0) {
                if (threadIdx.x == 0) *a.diverged_epoch = a.epoch;
                break;
            }
            if (threadIdx.x == 0) epoch_total = madd_rn(epoch_total, S.scal[1], (double)nb);
            const double lr = a.lr;
            for_each_owned(g, [&](int p, double& acc) {
                const double wv = get_smem_param(S, p);
                set_smem_param(S, p, (double)__double2float_rn(__dsub_rn(wv, __dmul_rn(lr, acc))));
            });
            zero_grads(g);
            __syncthreads();
        } else {
            // ---- per-CTA partials -> deterministic cross-CTA reduction
            double* part = a.partials + (size_t)blockIdx.x * (NP + 1);
            for_each_owned(g, [&](int p, double& acc) { part[p] = acc; });
            if (threadIdx.x == 0) part[NP] = g.loss;
            grid_barrier(a.bar, bar_target);
            if (threadIdx.x == 0) {
                double tot = 0.0;
                for (int c = 0; c < (int)gridDim.x; ++c)
                    tot = __dadd_rn(tot, __ldcg(a.partials + (size_t)c * (NP + 1) + NP));
                const double loss = __ddiv_rn(tot, (double)nb);
                S.scal[1] = loss;
                S.scal[2] = isfinite(loss) ? 0.0 : 1.0;
            }
            __syncthreads();
            if (S.scal[2] != 0.0) {
                if (blockIdx.x == 0 && threadIdx.x == 0) *a.diverged_epoch = a.epoch;
                break;
            }
            if (threadIdx.x == 0) epoch_total = madd_rn(epoch_total, S.scal[1], (double)nb);
            const int chunk = (NP + gridDim.x - 1) / gridDim.x;
            const int p_lo = blockIdx.x * chunk, p_hi = min(NP, p_lo + chunk);
            for (int p = p_lo + threadIdx.x; p < p_hi; p += blockDim.x) {
                double gs = 0.0;
                for (int c = 0; c < (int)gridDim.x; ++c)
                    gs = __dadd_rn(gs, __ldcg(a.partials + (size_t)c * (NP + 1) + p));
                const double wv = get_smem_param(S, p);
                a.params[p] = __double2float_rn(__dsub_rn(wv, __dmul_rn(a.lr, gs)));
            }
            grid_barrier(a.bar, bar_target);
            for (int t = threadIdx.x; t < NP; t += blockDim.x) set_smem_param(S, t, (double)__ldcg(a.params + t));
            zero_grads(g);
            __syncthreads();
        }
    }
    // epoch loss = total / n (policy.cpp:334); params back to global
    if (blockIdx.x == 0 && threadIdx.x == 0 && *a.diverged_epoch < 0)
        a.epoch_loss[a.epoch] = __ddiv_rn(epoch_total, (double)a.n);
    if (single) {
        __syncthreads();
        for (int t = threadIdx.x; t < NP; t += blockDim.x) a.params[t] = (float)get_smem_param(S, t);
    }
}

// Data-parallel path: one step's per-CTA partials only.
__global__ void __launch_bounds__(TRAIN_BLOCK, 1) train_partial_kernel(TrainArgs a, long step) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TrainSmem& S = *reinterpret_cast<TrainSmem*>(smem_raw);
    if (*a.diverged_epoch >= 0) return;
    load_train_weights(S, a.params);
    __syncthreads();
    GradRegs g;
    zero_grads(g);
    size_t nb;
    run_step_tiles(S, g, a, step, nb);
    double* part = a.partials + (size_t)blockIdx.x * (NP + 1);
    for_each_owned(g, [&](int p, double& acc) { part[p] = acc; });
    if (threadIdx.x == 0) part[NP] = g.loss;
}

// Sum per-CTA partials in CTA order into red[NP+1].
__global__ void reduce_partials_kernel(const double* __restrict__ partials, int nctas,
                                       double* __restrict__ red, const int* __restrict__ diverged) {
    if (*diverged >= 0) return;
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p > NP) return;
    double s = 0.0;
    for (int c = 0; c < nctas; ++c) s = __dadd_rn(s, partials[(size_t)c * (NP + 1) + p]);
    red[p] = s;
}

// SGD update from an (all-reduced) gradient + loss total; tracks epoch loss.
__global__ void apply_update_kernel(float* __restrict__ params, const double* __restrict__ red,
                                    double lr, size_t nb, int epoch, int* __restrict__ diverged,
                                    double* __restrict__ epoch_acc) {
    if (*diverged >= 0) return;
    const double loss = __ddiv_rn(red[NP], (double)nb);
    if (!isfinite(loss)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) *diverged = epoch;
        return;
    }
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < NP) params[p] = __double2float_rn(__dsub_rn((double)params[p], __dmul_rn(lr, red[p])));
    if (p == 0) *epoch_acc = madd_rn(*epoch_acc, loss, (double)nb);
}

__global__ void finish_epoch_kernel(const double* __restrict__ epoch_acc, size_t n, int epoch,
                                    const int* __restrict__ diverged, double* __restrict__ out) {
    if (*diverged >= 0) return;
    out[epoch] = __ddiv_rn(*epoch_acc, (double)n);
}

// ------------------------------------------------------ loss / gradient API
// batch_kl_loss / batch_kl_gradient for one batch (rows 0..n-1 in order):
// identical code path as fit with order = identity and a single step.
__global__ void __launch_bounds__(TRAIN_BLOCK, 1)
batch_grad_kernel(TrainArgs a, double* __restrict__ grad_out, double* __restrict__ loss_out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TrainSmem& S = *reinterpret_cast<TrainSmem*>(smem_raw);
    load_train_weights(S, a.params);
    __syncthreads();
    GradRegs g;
    zero_grads(g);
    size_t nb;
    run_step_tiles(S, g, a, 0, nb);
    for_each_owned(g, [&](int p, double& acc) { grad_out[p] = acc; });
    if (threadIdx.x == 0) *loss_out = __ddiv_rn(g.loss, (double)nb);
}

}  // namespace gbxcu
