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
//   F3 logits, softmax, KL, d3 = p (ln(p^/t^) - L) / |b|   (2 threads per record)
//   B1 d2[r][k]  = d3[r][0] w2[0][k] + d3[r][1] w2[1][k], masked by h2 > 0
//   B2 d1[r][j]  = sum_k d2[r][k] w1[k][j], masked by h1 > 0
//   G  gw2/gw1/gw0/gb* += per-record outer products, K = records in batch order
// Gradient accumulators are owned by threads (registers) across all tiles of a
// step, so a 1-CTA step reproduces the reference's per-parameter left fold bit
// for bit (up to exp/log ulps). Steps spread over several CTAs run on the FP64
// tensor cores instead (k_train_tc.cu).
//
// The records of the NEXT tile (possibly of the next step — the epoch's
// permutation is known up front) are gathered with cp.async into a second
// staging buffer while the current tile computes.
//
// Kernels
//   train_epoch_kernel<TB>  : one launch = one epoch on one GPU, one CTA
//                             (batches of <= 32 records per rank: the
//                             reference's default and its bit-exact regime).
//   train_partial_kernel<TB>: one step's partials on one CTA (data-parallel
//                             path; NCCL all-reduce and update follow).
//   batch_grad_kernel       : batch_kl_loss / batch_kl_gradient.
#include <cstddef>

#include "common.cuh"
#include "kernels.h"

namespace gbxcu {

#ifdef GBX_PHASE_TIMING
// Debug build only (tools/phase_timing.sh): per-phase cycle totals of CTA 0.
__device__ unsigned long long g_phase_cycles[16];
__device__ unsigned long long g_phase_t;
#define PHASE_MARK(i)                                                          \
    do {                                                                       \
        if (threadIdx.x == 0 && blockIdx.x == 0) {                             \
            const unsigned long long t_ = clock64();                           \
            g_phase_cycles[i] += t_ - g_phase_t;                               \
            g_phase_t = t_;                                                    \
        }                                                                      \
    } while (0)
#else
#define PHASE_MARK(i) ((void)0)
#endif

constexpr int NT = TRAIN_BLOCK;  // 512 threads
constexpr int NW = NT / 32;      // 16 warps

// Weight replicas are row-major with odd row strides (in 8-byte words), so a
// warp reading one column across 32 rows, or one row across 32 columns, hits
// 32 distinct banks: no transposed copies are needed and the owner-computes
// SGD update writes conflict-free.
constexpr int W0S = F + 1;   // 45
constexpr int W1S = H1 + 1;  // 65
// h2/d2 rows are also read/written record-parallel (F3: lanes = records), so
// their stride is padded off the 32-word period; 34 keeps 16-byte alignment
// for the double2 row reads of B2.
constexpr int H2S = H2 + 2;  // 34

template <int TB>
struct TrainSmem {
    double w0[H1 * W0S];  // [j][i], stride 45
    double w1[H2 * W1S];  // [k][j], stride 65
    double w2[A * H2];    // [a][k]
    double b0[H1];
    double b1[H2];
    double b2[A];
    double x[TB * F];    // [r][i]
    double h1[TB * H1];  // [r][j]
    double h2[TB * H2S]; // [r][k], stride 34
    double d2[TB * H2S]; // [r][k], stride 34
    double d1[TB * H1];  // [r][j]
    double d3[TB * 2];
    double tgt[TB * 2];
    double kl[TB];
    uint32_t ord[2][TB];        // record indices of the next two tiles (cp.async ring)
    double stage_t[2][TB * 2];  // cp.async staging: targets
    float stage_f[2][TB * F];   // cp.async staging: raw fp32 features
    double scal[4];             // [1] batch loss, [2] diverged flag
};

template <int TB>
constexpr bool smem_aligned() {
    return offsetof(TrainSmem<TB>, x) % 16 == 0 && offsetof(TrainSmem<TB>, h1) % 16 == 0 &&
           offsetof(TrainSmem<TB>, d2) % 16 == 0 && offsetof(TrainSmem<TB>, d1) % 16 == 0 &&
           offsetof(TrainSmem<TB>, stage_t) % 16 == 0 && offsetof(TrainSmem<TB>, stage_f) % 16 == 0;
}
static_assert(smem_aligned<32>() && smem_aligned<64>(), "16-byte aligned smem arrays");

size_t train_smem_bytes(int tb) {
    return tb == 32 ? sizeof(TrainSmem<32>) : sizeof(TrainSmem<64>);
}

// ----------------------------------------------------------- cp.async
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
                 "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// ------------------------------------------------------------ weights
template <int TB>
__device__ __forceinline__ void set_smem_param(TrainSmem<TB>& S, int p, double v) {
    if (p < OFF_B0) { const int j = p / F, i = p - j * F; S.w0[j * W0S + i] = v; }
    else if (p < OFF_W1) S.b0[p - OFF_B0] = v;
    else if (p < OFF_B1) {
        const int t = p - OFF_W1, k = t >> 6, j = t & 63;
        S.w1[k * W1S + j] = v;
    } else if (p < OFF_W2) S.b1[p - OFF_B1] = v;
    else if (p < OFF_B2) S.w2[p - OFF_W2] = v;
    else S.b2[p - OFF_B2] = v;
}

template <int TB>
__device__ __forceinline__ double get_smem_param(const TrainSmem<TB>& S, int p) {
    if (p < OFF_B0) { const int j = p / F, i = p - j * F; return S.w0[j * W0S + i]; }
    if (p < OFF_W1) return S.b0[p - OFF_B0];
    if (p < OFF_B1) { const int t = p - OFF_W1; return S.w1[(t >> 6) * W1S + (t & 63)]; }
    if (p < OFF_W2) return S.b1[p - OFF_B1];
    if (p < OFF_B2) return S.w2[p - OFF_W2];
    return S.b2[p - OFF_B2];
}

// All threads: fp32 master params (global) -> fp64 smem replicas, float2 loads
// (NP is even; the buffer is 8-byte aligned).
template <int TB>
__device__ void load_train_weights(TrainSmem<TB>& S, const float* __restrict__ p, bool coherent) {
    const float2* p2 = reinterpret_cast<const float2*>(p);
    constexpr int N2 = NP / 2;
    constexpr int PER = (N2 + NT - 1) / NT;
    float2 v[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const int t = threadIdx.x + q * NT;
        if (t < N2) v[q] = coherent ? __ldcg(p2 + t) : __ldg(p2 + t);
    }
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const int t = threadIdx.x + q * NT;
        if (t < N2) {
            set_smem_param(S, 2 * t, (double)v[q].x);
            set_smem_param(S, 2 * t + 1, (double)v[q].y);
        }
    }
}

// ------------------------------------------------- gradient ownership
// gw0: lane owns columns j = lane, lane+32; warp w owns inputs i = 2w, 2w+1 and,
//      for w < 12, i = 32 + w (44 = 2*16 + 12): 4 or 6 accumulators.
// gw1: warp w owns rows k = 2w, 2w+1 at columns j = lane, lane+32.
// gb0: warp 12 (one of the lighter warps) owns j = lane, lane+32.
// extras (gx): tid 320..351 gb1[k], 352..415 gw2[a][k], 416..417 gb2[a];
// tid NT-1 keeps the running KL sum.
struct GradRegs {
    double g0[3][2];  // [i-slot][j-slot]
    double g1[2][2];
    double gb0[2];
    double gx;
    double loss;
};

__device__ __forceinline__ int g0_col(int w, int m) { return m < 2 ? 2 * w + m : 32 + w; }
__device__ __forceinline__ int g0_slots(int w) { return w < F - 32 ? 3 : 2; }

__device__ __forceinline__ void zero_grads(GradRegs& g) {
#pragma unroll
    for (int m = 0; m < 3; ++m) g.g0[m][0] = g.g0[m][1] = 0.0;
    g.g1[0][0] = g.g1[0][1] = g.g1[1][0] = g.g1[1][1] = 0.0;
    g.gb0[0] = g.gb0[1] = 0.0;
    g.gx = 0.0;
    g.loss = 0.0;
}

template <typename Fn>
__device__ __forceinline__ void for_each_owned(GradRegs& g, Fn fn) {
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
#pragma unroll
    for (int m = 0; m < 3; ++m) {
        if (m < g0_slots(w)) {
            const int i = g0_col(w, m);
            fn(OFF_W0 + lane * F + i, g.g0[m][0]);
            fn(OFF_W0 + (lane + 32) * F + i, g.g0[m][1]);
        }
    }
#pragma unroll
    for (int kk = 0; kk < 2; ++kk)
#pragma unroll
        for (int q = 0; q < 2; ++q) fn(OFF_W1 + (2 * w + kk) * H1 + lane + 32 * q, g.g1[kk][q]);
    if (w == 12) {
        fn(OFF_B0 + lane, g.gb0[0]);
        fn(OFF_B0 + lane + 32, g.gb0[1]);
    }
    if (tid >= 320 && tid < 352) fn(OFF_B1 + tid - 320, g.gx);
    else if (tid >= 352 && tid < 416) fn(OFF_W2 + tid - 352, g.gx);
    else if (tid >= 416 && tid < 418) fn(OFF_B2 + tid - 416, g.gx);
}

// w = float(double(w) - lr * g) (policy.cpp:329-331), kept as fp64 in smem.
__device__ __forceinline__ double sgd(double w, double lr, double g) {
    return (double)__double2float_rn(__dsub_rn(w, __dmul_rn(lr, g)));
}

// 1-CTA step: every owner updates its parameters in the smem replica directly
// (w0 rows have odd stride 45, so the column-parallel writes are conflict-free).
template <int TB>
__device__ __forceinline__ void sgd_update_owned(TrainSmem<TB>& S, const GradRegs& g, double lr) {
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
#pragma unroll
    for (int m = 0; m < 3; ++m) {
        if (m < g0_slots(w)) {
            const int i = g0_col(w, m);
            double* a = S.w0 + lane * W0S + i;
            double* b = S.w0 + (lane + 32) * W0S + i;
            *a = sgd(*a, lr, g.g0[m][0]);
            *b = sgd(*b, lr, g.g0[m][1]);
        }
    }
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
        double* row = S.w1 + (2 * w + kk) * W1S;
        row[lane] = sgd(row[lane], lr, g.g1[kk][0]);
        row[lane + 32] = sgd(row[lane + 32], lr, g.g1[kk][1]);
    }
    if (w == 12) {
        S.b0[lane] = sgd(S.b0[lane], lr, g.gb0[0]);
        S.b0[lane + 32] = sgd(S.b0[lane + 32], lr, g.gb0[1]);
    }
    if (tid >= 320 && tid < 352) S.b1[tid - 320] = sgd(S.b1[tid - 320], lr, g.gx);
    else if (tid >= 352 && tid < 416) S.w2[tid - 352] = sgd(S.w2[tid - 352], lr, g.gx);
    else if (tid >= 416 && tid < 418) S.b2[tid - 416] = sgd(S.b2[tid - 416], lr, g.gx);
}

// ------------------------------------------------------------ tiling
// Records of step `step` handled by CTA `cta` of `nctas` on rank `rank`:
// equal contiguous slices of the global batch, rank-major then CTA-major.
// n < 2^31 and batch < 2^31 are validated on the host, so 32-bit math suffices.
__device__ __forceinline__ void step_slice(const TrainArgs& a, long step, int cta, int nctas,
                                           size_t& lo, size_t& hi, size_t& nb) {
    const uint32_t n = (uint32_t)a.n, batch = (uint32_t)a.batch;
    const uint32_t start = (uint32_t)step * batch;
    const uint32_t stop = min(n, start + batch);
    const uint32_t nbu = stop - start;
    const uint32_t per_rank = (nbu + a.nranks - 1) / (uint32_t)a.nranks;
    const uint32_t r_lo = min(stop, start + (uint32_t)a.rank * per_rank);
    const uint32_t r_hi = min(stop, r_lo + per_rank);
    const uint32_t per_cta = (r_hi - r_lo + nctas - 1) / (uint32_t)nctas;
    const uint32_t l = min(r_hi, r_lo + (uint32_t)cta * per_cta);
    lo = l;
    hi = min(r_hi, l + per_cta);
    nb = nbu;
}

// Next tile of this CTA after (step, r0) within steps < step_end. r0 == SIZE_MAX
// asks for the first tile of `step`.
template <int TB>
__device__ bool next_tile(const TrainArgs& a, long step_end, long& step, size_t& r0, int& nv) {
    size_t lo, hi, nb;
    if (r0 != (size_t)-1) {
        step_slice(a, step, blockIdx.x, gridDim.x, lo, hi, nb);
        if (r0 + TB < hi) {
            r0 += TB;
            nv = (int)min((size_t)TB, hi - r0);
            return true;
        }
        ++step;
    }
    for (; step < step_end; ++step) {
        step_slice(a, step, blockIdx.x, gridDim.x, lo, hi, nb);
        if (hi > lo) {
            r0 = lo;
            nv = (int)min((size_t)TB, hi - lo);
            return true;
        }
    }
    return false;
}

template <int TB>
__device__ void prefetch_tile(TrainSmem<TB>& S, int buf, const TrainArgs& a, size_t r0, int nv) {
    for (int t = threadIdx.x; t < TB * (F / 4); t += NT) {
        const int r = t / (F / 4), q = t - r * (F / 4);
        const float* src = a.feat;
        if (r < nv) src = a.feat + (size_t)a.order[r0 + r] * F + 4 * q;
        cp_async16(&S.stage_f[buf][r * F + 4 * q], src, r < nv ? 16 : 0);
    }
    if (threadIdx.x < TB) {
        const int r = threadIdx.x;
        const double* src = a.tgt;
        if (r < nv) src = a.tgt + 2 * (size_t)a.order[r0 + r];
        cp_async16(&S.stage_t[buf][2 * r], src, r < nv ? 16 : 0);
    }
    cp_async_commit();
}

// Epoch kernel ring: record indices of a tile two ahead, then its rows one
// ahead through the indices already in shared memory (the row gather issues
// without a dependent global load on the step's critical path).
template <int TB>
__device__ __forceinline__ void fetch_idx(TrainSmem<TB>& S, int slot, const TrainArgs& a, size_t r0, int nv) {
    if ((int)threadIdx.x < nv) {
        const unsigned d = (unsigned)__cvta_generic_to_shared(&S.ord[slot][threadIdx.x]);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(a.order + r0 + threadIdx.x)
                     : "memory");
    }
}
template <int TB>
__device__ __forceinline__ void fetch_rows(TrainSmem<TB>& S, int slot, const TrainArgs& a, int nv) {
    for (int t = threadIdx.x; t < TB * (F / 4); t += NT) {
        const int r = t / (F / 4), q = t - r * (F / 4);
        const float* src = a.feat;
        if (r < nv) src = a.feat + (size_t)S.ord[slot][r] * F + 4 * q;
        cp_async16(&S.stage_f[slot][r * F + 4 * q], src, r < nv ? 16 : 0);
    }
    if (threadIdx.x < TB) {
        const int r = threadIdx.x;
        const double* src = a.tgt;
        if (r < nv) src = a.tgt + 2 * (size_t)S.ord[slot][r];
        cp_async16(&S.stage_t[slot][2 * r], src, r < nv ? 16 : 0);
    }
}

// One tile: rows [0, nv) of the staged buffer `buf`; accumulates into g.
template <int TB>
__device__ void train_tile(TrainSmem<TB>& S, GradRegs& g, int buf, int nv, double inv_b) {
    constexpr int RPW = TB / NW;  // rows per warp in the row-parallel phases
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;

    // ---- P0: staged fp32 -> fp64 tile
    for (int t = tid; t < TB * F; t += NT) S.x[t] = (double)S.stage_f[buf][t];
    if (tid < 2 * TB) S.tgt[tid] = S.stage_t[buf][tid];
    __syncthreads();

    PHASE_MARK(0);
    // ---- F1: lanes <-> j (lane, lane+32), warp <-> rows
    {
        double acc[RPW][2];
        const double bA = S.b0[lane], bB = S.b0[lane + 32];
#pragma unroll
        for (int rr = 0; rr < RPW; ++rr) { acc[rr][0] = bA; acc[rr][1] = bB; }
        const double* xb = S.x + (RPW * w) * F;
#pragma unroll 2
        for (int i = 0; i < F; i += 2) {
            const double* wa = S.w0 + lane * W0S + i;
            const double* wb = S.w0 + (lane + 32) * W0S + i;
            const double wA0 = wa[0], wB0 = wb[0], wA1 = wa[1], wB1 = wb[1];
#pragma unroll
            for (int rr = 0; rr < RPW; ++rr) {
                const double2 xv = *reinterpret_cast<const double2*>(xb + rr * F + i);
                // fp32 x fp32 products are exact in fp64, so DFMA == mul-then-add
                acc[rr][0] = fma(wA0, xv.x, acc[rr][0]);
                acc[rr][1] = fma(wB0, xv.x, acc[rr][1]);
                acc[rr][0] = fma(wA1, xv.y, acc[rr][0]);
                acc[rr][1] = fma(wB1, xv.y, acc[rr][1]);
            }
        }
#pragma unroll
        for (int rr = 0; rr < RPW; ++rr) {
            double* hr = S.h1 + (RPW * w + rr) * H1;
            hr[lane] = acc[rr][0] > 0.0 ? acc[rr][0] : 0.0;
            hr[lane + 32] = acc[rr][1] > 0.0 ? acc[rr][1] : 0.0;
        }
    }
    __syncthreads();

    PHASE_MARK(1);
    // ---- F2: lanes <-> k, warp <-> rows
    {
        double acc[RPW];
        const double b = S.b1[lane];
#pragma unroll
        for (int rr = 0; rr < RPW; ++rr) acc[rr] = b;
        const double* hb = S.h1 + (RPW * w) * H1;
#pragma unroll 4
        for (int j = 0; j < H1; j += 2) {
            const double w0 = S.w1[lane * W1S + j], w1 = S.w1[lane * W1S + j + 1];
#pragma unroll
            for (int rr = 0; rr < RPW; ++rr) {
                const double2 hv = *reinterpret_cast<const double2*>(hb + rr * H1 + j);
                acc[rr] = madd_rn(acc[rr], w0, hv.x);
                acc[rr] = madd_rn(acc[rr], w1, hv.y);
            }
        }
#pragma unroll
        for (int rr = 0; rr < RPW; ++rr)
            S.h2[(RPW * w + rr) * H2S + lane] = acc[rr] > 0.0 ? acc[rr] : 0.0;
    }
    __syncthreads();

    PHASE_MARK(2);
    // ---- F3: thread (r, a) computes logit a, then softmax/KL/d3 with its pair
    if (tid < 2 * TB) {
        const int r = tid >> 1, a = tid & 1;
        double l = S.b2[a];
        const double* h = S.h2 + r * H2S;
        const double* wr = S.w2 + a * H2;
#pragma unroll 8
        for (int k = 0; k < H2; ++k) l = madd_rn(l, wr[k], h[k]);
        const double lo = __shfl_xor_sync(0xffffffffu, l, 1);
        const double l0 = a ? lo : l, l1 = a ? l : lo;
        const double m = l0 < l1 ? l1 : l0;  // std::max(l0, l1)
        const double e = exp(__dsub_rn(l, m));
        const double eo = __shfl_xor_sync(0xffffffffu, e, 1);
        const double s = a ? __dadd_rn(eo, e) : __dadd_rn(e, eo);  // e0 + e1
        const double p = __ddiv_rn(e, s);
        const double pc = clampp(p);
        const double tc = clampp(S.tgt[2 * r + a]);
        const double lr = log(__ddiv_rn(pc, tc));
        const double term = __dmul_rn(pc, lr);
        const double to = __shfl_xor_sync(0xffffffffu, term, 1);
        const double loss = __dadd_rn(__dadd_rn(0.0, a ? to : term), a ? term : to);
        const bool valid = r < nv;
        if (a == 0) S.kl[r] = valid ? loss : 0.0;
        const double d3 = valid ? __dmul_rn(__dmul_rn(p, __dsub_rn(lr, loss)), inv_b) : 0.0;
        S.d3[2 * r + a] = d3;
        // ---- B1 (same pair): d2[r][k] = (0 + d3_0 w2_0k) + d3_1 w2_1k, masked by
        //      h2 > 0; thread a covers k in [16a, 16a+16)
        const double d3o = __shfl_xor_sync(0xffffffffu, d3, 1);
        const double d30 = a ? d3o : d3, d31 = a ? d3 : d3o;
#pragma unroll
        for (int kk = 0; kk < H2 / 2; ++kk) {
            const int k = (H2 / 2) * a + kk;
            double d = madd_rn(0.0, d30, S.w2[k]);
            d = madd_rn(d, d31, S.w2[H2 + k]);
            S.d2[r * H2S + k] = h[k] <= 0.0 ? 0.0 : d;
        }
    }
    __syncthreads();

    PHASE_MARK(3);
    // ---- B2: d1[r][j] = sum_k d2[r][k] w1[k][j] (masked by h1 > 0)
    //      + gw1 / gb1 / gw2 / gb2 / KL-sum accumulation (need only d2, d3, h1, h2)
    {
        double acc[RPW][2];
#pragma unroll
        for (int rr = 0; rr < RPW; ++rr) acc[rr][0] = acc[rr][1] = 0.0;
        const double* db = S.d2 + (RPW * w) * H2S;
#pragma unroll 4
        for (int k = 0; k < H2; k += 2) {
            const double* wk = S.w1 + k * W1S;
            const double wA0 = wk[lane], wB0 = wk[lane + 32];
            const double wA1 = wk[W1S + lane], wB1 = wk[W1S + lane + 32];
#pragma unroll
            for (int rr = 0; rr < RPW; ++rr) {
                const double2 dv = *reinterpret_cast<const double2*>(db + rr * H2S + k);
                // a zero d2 adds a signed zero: a no-op, matching the reference's
                // `continue` on zero rows (policy.cpp:247)
                acc[rr][0] = madd_rn(acc[rr][0], dv.x, wA0);
                acc[rr][1] = madd_rn(acc[rr][1], dv.x, wB0);
                acc[rr][0] = madd_rn(acc[rr][0], dv.y, wA1);
                acc[rr][1] = madd_rn(acc[rr][1], dv.y, wB1);
            }
        }
#pragma unroll
        for (int rr = 0; rr < RPW; ++rr) {
            const int r = RPW * w + rr;
            S.d1[r * H1 + lane] = S.h1[r * H1 + lane] <= 0.0 ? 0.0 : acc[rr][0];
            S.d1[r * H1 + lane + 32] = S.h1[r * H1 + lane + 32] <= 0.0 ? 0.0 : acc[rr][1];
        }
        // gw1[2w+kk][lane+32q] += d2[r][2w+kk] * h1[r][lane+32q], r in batch order
#pragma unroll 4
        for (int r = 0; r < nv; ++r) {
            const double2 dk = *reinterpret_cast<const double2*>(S.d2 + r * H2S + 2 * w);
            const double hA = S.h1[r * H1 + lane], hB = S.h1[r * H1 + lane + 32];
            g.g1[0][0] = madd_rn(g.g1[0][0], dk.x, hA);
            g.g1[0][1] = madd_rn(g.g1[0][1], dk.x, hB);
            g.g1[1][0] = madd_rn(g.g1[1][0], dk.y, hA);
            g.g1[1][1] = madd_rn(g.g1[1][1], dk.y, hB);
        }
        if (tid >= 320 && tid < 352) {
            const int k = tid - 320;
            for (int r = 0; r < nv; ++r) g.gx = __dadd_rn(g.gx, S.d2[r * H2S + k]);
        } else if (tid >= 352 && tid < 416) {
            const int a = (tid - 352) >> 5, k = (tid - 352) & 31;
            for (int r = 0; r < nv; ++r) g.gx = madd_rn(g.gx, S.d3[2 * r + a], S.h2[r * H2S + k]);
        } else if (tid >= 416 && tid < 418) {
            const int a = tid - 416;
            for (int r = 0; r < nv; ++r) g.gx = __dadd_rn(g.gx, S.d3[2 * r + a]);
        } else if (tid == NT - 1) {
            for (int r = 0; r < nv; ++r) g.loss = __dadd_rn(g.loss, S.kl[r]);
            // divergence flag of the step so far (loss = sum / |b| is finite iff
            // the sum is): read after the tile's closing barrier
            S.scal[2] = isfinite(g.loss) ? 0.0 : 1.0;
        }
    }
    __syncthreads();

    PHASE_MARK(4);
    // ---- G0: gw0[j][i] += d1[r][j] * x[r][i] (j = lane, lane+32; i = warp's
    //      columns), gb0[j] += d1[r][j] on warp 12; records in batch order
    {
        const int i0 = 2 * w, i2 = 32 + w;
        const bool three = w < F - 32;
#pragma unroll 2
        for (int r = 0; r < nv; ++r) {
            const double2 xp = *reinterpret_cast<const double2*>(S.x + r * F + i0);
            const double da = S.d1[r * H1 + lane], db = S.d1[r * H1 + lane + 32];
            g.g0[0][0] = madd_rn(g.g0[0][0], da, xp.x);
            g.g0[0][1] = madd_rn(g.g0[0][1], db, xp.x);
            g.g0[1][0] = madd_rn(g.g0[1][0], da, xp.y);
            g.g0[1][1] = madd_rn(g.g0[1][1], db, xp.y);
            if (three) {
                const double x2 = S.x[r * F + i2];
                g.g0[2][0] = madd_rn(g.g0[2][0], da, x2);
                g.g0[2][1] = madd_rn(g.g0[2][1], db, x2);
            }
            if (w == 12) {
                g.gb0[0] = __dadd_rn(g.gb0[0], da);
                g.gb0[1] = __dadd_rn(g.gb0[1], db);
            }
        }
    }
    __syncthreads();
    PHASE_MARK(5);
}

// Deterministic fixed-shape warp sum of per-lane partials (lane 0 holds it).
__device__ __forceinline__ double warp_tree_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, o));
    return v;
}

// Sum of partials[c][p] over c < G with a fixed association (per-lane strided
// left fold, then a shuffle-down tree). Called by a full warp; lane 0 result.
__device__ __forceinline__ double reduce_over_ctas(const double* __restrict__ partials, int G,
                                                   int p, int lane) {
    double v = 0.0;
    for (int c = lane; c < G; c += 32) v = __dadd_rn(v, __ldcg(partials + (size_t)c * PSTR + p));
    return warp_tree_sum(v);
}

template <int TB>
__global__ void __launch_bounds__(NT, 1) train_epoch_kernel(TrainArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TrainSmem<TB>& S = *reinterpret_cast<TrainSmem<TB>*>(smem_raw);
    if (*a.diverged_epoch >= 0) return;  // an earlier epoch diverged
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const long n_steps = (long)((a.n + a.batch - 1) / a.batch);

    // Ring (tile k): rows of tile k in stage[k & 1] (fetched during tile
    // k - 1), indices of tile k + 1 in ord[(k + 1) & 1]. Cursors: c1 = tile
    // k + 1, c2 = tile k + 2.
    long s1 = 0, s2 = 0;
    size_t r1 = (size_t)-1, r2 = 0;
    int n1 = 0, n2 = 0;
    bool h1 = next_tile<TB>(a, n_steps, s1, r1, n1);  // tile 0
    if (h1) fetch_idx(S, 0, a, r1, n1);
    s2 = s1;
    r2 = r1;
    bool h2 = h1 && next_tile<TB>(a, n_steps, s2, r2, n2);  // tile 1
    if (h2) fetch_idx(S, 1, a, r2, n2);
    cp_async_commit();
    load_train_weights(S, a.params, false);
    cp_async_wait_all();
    __syncthreads();
    if (h1) fetch_rows(S, 0, a, n1);
    cp_async_commit();
    h1 = h2; s1 = s2; r1 = r2; n1 = n2;  // c1 <- tile 1, c2 <- tile 2
    s2 = s1; r2 = r1;
    h2 = h1 && next_tile<TB>(a, n_steps, s2, r2, n2);
    GradRegs g;
    zero_grads(g);
    double epoch_total = 0.0;  // thread NT - 1 (it holds the loss sums)
    int k = 0;

    for (long step = 0; step < n_steps; ++step) {
        size_t lo, hi, nb;
        step_slice(a, step, 0, 1, lo, hi, nb);
        const double inv_b = 1.0 / (double)nb;  // batch_kl_gradient's 1/|b| (global batch)
        for (size_t r0 = lo; r0 < hi; r0 += TB, ++k) {
            const int nv = (int)min((size_t)TB, hi - r0);
            PHASE_MARK(6);
            cp_async_wait_all();  // this thread's copies: tile k's rows, tile k+1's indices
            __syncthreads();
            if (h1) fetch_rows(S, (k + 1) & 1, a, n1);  // rows of tile k+1
            if (h2) fetch_idx(S, k & 1, a, r2, n2);     // indices of tile k+2
            cp_async_commit();
            h1 = h2; s1 = s2; r1 = r2; n1 = n2;
            if (h2) h2 = next_tile<TB>(a, n_steps, s2, r2, n2);
            PHASE_MARK(7);
            train_tile<TB>(S, g, k & 1, nv, inv_b);
        }
        // loss = (sum of per-record KL, batch order) / |b|  (policy.cpp:194-201);
        // its finiteness was flagged in B2, before the tile's closing barrier
        if (S.scal[2] != 0.0) {
            if (tid == 0) *a.diverged_epoch = a.epoch;
            break;
        }
        if (tid == NT - 1) epoch_total = madd_rn(epoch_total, __ddiv_rn(g.loss, (double)nb), (double)nb);
        sgd_update_owned(S, g, a.lr);
        zero_grads(g);
        __syncthreads();
    }
    cp_async_wait_all();
    // epoch loss = total / n (policy.cpp:334); params back to global
    if (tid == NT - 1 && *a.diverged_epoch < 0)
        a.epoch_loss[a.epoch] = __ddiv_rn(epoch_total, (double)a.n);
    __syncthreads();
    for (int t = tid; t < NP; t += NT) a.params[t] = (float)get_smem_param(S, t);
}

// Data-parallel path: one step's per-CTA partials only.
template <int TB>
__global__ void __launch_bounds__(NT, 1) train_partial_kernel(TrainArgs a, long step) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TrainSmem<TB>& S = *reinterpret_cast<TrainSmem<TB>*>(smem_raw);
    if (*a.diverged_epoch >= 0) return;
    size_t lo, hi, nb;
    step_slice(a, step, blockIdx.x, gridDim.x, lo, hi, nb);
    if (hi > lo) prefetch_tile<TB>(S, 0, a, lo, (int)min((size_t)TB, hi - lo));
    load_train_weights(S, a.params, false);
    GradRegs g;
    zero_grads(g);
    const double inv_b = 1.0 / (double)nb;
    int buf = 0;
    for (size_t r0 = lo; r0 < hi; r0 += TB) {
        const int nv = (int)min((size_t)TB, hi - r0);
        cp_async_wait_all();
        __syncthreads();
        const int cur = buf;
        buf ^= 1;
        if (r0 + TB < hi) prefetch_tile<TB>(S, buf, a, r0 + TB, (int)min((size_t)TB, hi - r0 - TB));
        train_tile<TB>(S, g, cur, nv, inv_b);
    }
    double* part = a.partials + (size_t)blockIdx.x * PSTR;
    for_each_owned(g, [&](int p, double& acc) { part[p] = acc; });
    if (threadIdx.x == NT - 1) part[NP] = g.loss;
}

// Sum per-CTA partials (fixed tree) into red[NP+1]; one warp per entry.
__global__ void reduce_partials_kernel(const double* __restrict__ partials, int nctas,
                                       double* __restrict__ red, const int* __restrict__ diverged) {
    if (*diverged >= 0) return;
    const int p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (p > NP) return;
    const double s = reduce_over_ctas(partials, nctas, p, threadIdx.x & 31);
    if ((threadIdx.x & 31) == 0) red[p] = s;
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

// batch_kl_loss / batch_kl_gradient for one batch (rows 0..n-1 in order):
// fit's tile code with order = identity and a single 1-CTA step.
__global__ void __launch_bounds__(NT, 1)
batch_grad_kernel(TrainArgs a, double* __restrict__ grad_out, double* __restrict__ loss_out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TrainSmem<64>& S = *reinterpret_cast<TrainSmem<64>*>(smem_raw);
    load_train_weights(S, a.params, false);
    GradRegs g;
    zero_grads(g);
    const double inv_b = 1.0 / (double)a.n;
    for (size_t r0 = 0; r0 < a.n; r0 += 64) {
        const int nv = (int)min((size_t)64, a.n - r0);
        __syncthreads();
        prefetch_tile<64>(S, 0, a, r0, nv);
        cp_async_wait_all();
        __syncthreads();
        train_tile<64>(S, g, 0, nv, inv_b);
    }
    for_each_owned(g, [&](int p, double& acc) { grad_out[p] = acc; });
    if (threadIdx.x == NT - 1) *loss_out = __ddiv_rn(g.loss, (double)a.n);
}

template __global__ void train_epoch_kernel<32>(TrainArgs);
template __global__ void train_epoch_kernel<64>(TrainArgs);
template __global__ void train_partial_kernel<32>(TrainArgs, long);
template __global__ void train_partial_kernel<64>(TrainArgs, long);

}  // namespace gbxcu

#ifdef GBX_PHASE_TIMING
extern "C" int gbxcu_debug_phase_cycles(unsigned long long* out, int reset) {
    if (cudaMemcpyFromSymbol(out, gbxcu::g_phase_cycles, sizeof(unsigned long long) * 16) != cudaSuccess)
        return 3;
    if (reset) {
        unsigned long long z[16] = {};
        cudaMemcpyToSymbol(gbxcu::g_phase_cycles, z, sizeof(z));
    }
    return 0;
}
#endif
