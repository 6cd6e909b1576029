// k_train_tc.cu — multi-CTA fused train epoch (K1, throughput regime) on the
// FP64 tensor cores (DMMA m8n8k4), sm_100a.
//
// Replaces fit's inner loop (proj/src/policy.cpp:316-333) when a step's batch
// is spread over G > 1 CTAs: batch_kl_loss / batch_kl_gradient (forward +
// analytic backward, :29-55, :209-279) and the SGD update
// w = float(double(w) - lr * g) (:328-332).
//
// Numerics: fp32 parameters, fp64 arithmetic everywhere (as the reference),
// but the contractions run as fp64 MMA (fused multiply-add, tensor-core
// summation order) instead of the reference's sequential mul-then-add. A
// multi-CTA step already re-associates the gradient sum across CTAs, so this
// path is graded by tolerance (<= 2 fp32 ulp per weight, losses rel 1e-12);
// the bit-exact 1-CTA path stays in k_train.cu.
//
// One tile = 8*MT records (MT m-tiles of 8). Per tile, all on DMMA:
//   F1  H1 = relu(X W0^T + b0)      M=8MT  N=64  K=44   (C initialised with b0)
//   F2  H2 = relu(H1 W1^T + b1)     M=8MT  N=32  K=64
//   F3  logits = H2 W2^T + b2       M=8MT  N=8(2) K=32  (warp w < MT owns m-tile w)
//       softmax / KL / d3 in the lanes holding each record's logits, then
//   B1  D2 = ([d3|0] [W2;0]) o [h2 > 0]   K=4 from the same lanes' registers
//   B2  D1 = (D2 W1) o [h1 > 0]     M=8MT  N=64  K=32
//   G1  [gW1|gb1] += D2^T [H1|1]    M=32   N=72  K=8MT (H1 column 64 == 1 gives gb1)
//   E   [gW2|gb2; .|KL] += U^T [H2|1]  M=8 N=40 K=8MT (U = [d3_0 d3_1 kl 0..])
//   G0  [gW0|gb0]^T += [X|1]^T D1   M=48   N=64  K=8MT (X column 44 == 1 gives gb0)
// Gradient accumulators (G1, E, G0) stay in registers across the tiles of a step.
// Operand layouts use row strides = 4 or 12 (mod 16) doubles, so every m8n8k4
// fragment load (row- or column-wise) is bank-conflict free.
//
// Step synchronisation (one arrival counter + data-flow words):
//   1. every CTA stores its gradient+loss partial (row of PSTR doubles) and
//      arrives on a monotonic counter (red.release); one thread per CTA polls
//      it (ld.acquire) while the other warps stage the next tile;
//   2. CTA c then reduces the contiguous slice
//      [c*chunk, (c+1)*chunk) of every partial plus the loss (fixed order:
//      8 CTA subsets x strided folds, then an in-order sum of the 8) — every
//      CTA reduces the loss identically, so all agree on divergence;
//   3. CTA c applies SGD to its slice and publishes each new parameter as a
//      64-bit word {tag, fp32 bits} (NCCL "LL" style: the tag validates the
//      value, single-copy atomic, no fence or flag round trip);
//   4. every CTA spins on the words of all parameters (one L2 round trip in
//      the common case) and rebuilds its fp64 shared-memory replicas.
// A producer cannot overwrite a partial / parameter word before every
// consumer has read it: its next write needs inputs that only exist after
// all consumers have moved on.
#include <cstddef>

#include "common.cuh"
#include "kernels.h"

namespace gbxcu {

#ifdef GBX_PHASE_TIMING
// Debug build only (tools/phase_timing.sh): per-phase cycle totals of CTA 0.
__device__ unsigned long long g_tc_phase[16];
__device__ unsigned long long g_tc_t;
__device__ unsigned long long g_tc_trace[8][160][6];  // steps 8..15: per-CTA globaltimer marks
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define TC_TRACE(step, k)                                                                      \
    do {                                                                                       \
        if (threadIdx.x == 0 && (step) >= 8 && (step) < 16 && blockIdx.x < 160)               \
            g_tc_trace[(step) - 8][blockIdx.x][k] = gtimer();                                  \
    } while (0)
#define TC_MARK(i)                                                                             \
    do {                                                                                       \
        if (threadIdx.x == 0 && blockIdx.x == 0) {                                             \
            const unsigned long long t_ = clock64();                                           \
            if ((i) >= 0) g_tc_phase[(i) < 0 ? 0 : (i)] += t_ - g_tc_t;                        \
            g_tc_t = t_;                                                                       \
        }                                                                                      \
    } while (0)
#else
#define TC_MARK(i) ((void)0)
#define TC_TRACE(step, k) ((void)0)
#endif

static_assert(PSTR >= NP + 1 && PSTR % 2 == 0, "partial rows hold NP params + loss, 16-B aligned");

namespace {

constexpr int NT = TRAIN_BLOCK;  // 512
constexpr int NW = NT / 32;      // 16 warps
constexpr int SX = 52;           // X  [r][i]: 44 features, col 44 = 1.0, 45..51 = 0
constexpr int SW0 = 44;          // W0 [j][i]
constexpr int SW1 = 68;          // W1 [k][j]
constexpr int SH1 = 68;          // H1, D1 [r][j]
constexpr int SH2 = 36;          // H2, D2 [r][k]: H2 col 32 = 1.0
constexpr int SU = 12;           // U [r][m]: d3_0, d3_1, kl, then zeros
constexpr double LN_PMIN = -16.11809565095832;        // ln(1e-7)
constexpr double LN_PMAX = -1.0000000494736474e-07;   // ln(double(1 - 1e-7))

template <int MT>
struct TcSmem {
    static constexpr int TB = 8 * MT;
    double w0[H1 * SW0];
    double w1[H2 * SW1];
    double w2[A * H2];
    double b0[H1];
    double b1[H2];
    double b2[A];
    double scal[2];
    double x[TB * SX];
    double h1[TB * SH1];
    double d1[TB * SH1];
    double h2[TB * SH2];
    double d2[TB * SH2];
    double u[TB * SU];
    double ltgt[TB * 2];         // ln(clamp(target)) per (record, action)
    double red[NT + 64];         // slice reduction: [source subset][element], then totals
    double adam[2][64];          // Adam m, v of this CTA's slice (kept on chip for the epoch)
    uint32_t ord[2][TB];         // record indices of the next two tiles (cp.async ring)
    double stage_t[2][TB * 2];   // cp.async staging: targets
    float stage_f[2][TB * F];    // cp.async staging: raw fp32 features
};

template <int MT>
constexpr bool tc_aligned() {
    return offsetof(TcSmem<MT>, x) % 16 == 0 && offsetof(TcSmem<MT>, h1) % 16 == 0 &&
           offsetof(TcSmem<MT>, stage_t) % 16 == 0 && offsetof(TcSmem<MT>, stage_f) % 16 == 0;
}
static_assert(tc_aligned<4>() && tc_aligned<7>(), "16-byte aligned smem arrays");

// D = A B + D for one 8x8x4 fp64 tile. Fragments (lane = 4g + t):
//   A[g][t] (row-major 8x4), B[t][g] (4x8), D[g][2t], D[g][2t+1].
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(d[0]), "+d"(d[1])
        : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
                 "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// Exchange accesses. Within one GPU (a single rank, or virtual ranks) they are
// GPU-scope; a real peer set spans GPUs of the NVLink domain and needs
// system scope (SYS), which is markedly more expensive.
template <bool SYS>
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    if (SYS) asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    else asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
template <bool SYS>
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    if (SYS) asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    else asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
template <bool SYS>
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
    if (SYS) asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
    else asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// LL pairs for the per-GPU sums of a peer set: a double travels as
// {tag | low 32 bits}, {tag | high 32 bits} in one 16-byte strong access
// (each 8-byte word is single-copy atomic and validates itself).
template <bool SYS>
__device__ __forceinline__ void ld_v2(const unsigned long long* p, unsigned long long& lo,
                                      unsigned long long& hi) {
    if (SYS)
        asm volatile("ld.relaxed.sys.global.v2.u64 {%0,%1}, [%2];" : "=l"(lo), "=l"(hi) : "l"(p) : "memory");
    else
        asm volatile("ld.relaxed.gpu.global.v2.u64 {%0,%1}, [%2];" : "=l"(lo), "=l"(hi) : "l"(p) : "memory");
}
template <bool SYS>
__device__ __forceinline__ void st_ll_pair(unsigned long long* p, double v, unsigned tag) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    const unsigned long long t = (unsigned long long)tag << 32;
    const unsigned long long lo = t | (b & 0xFFFFFFFFull), hi = t | (b >> 32);
    if (SYS)
        asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1,%2};" ::"l"(p), "l"(lo), "l"(hi) : "memory");
    else
        asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1,%2};" ::"l"(p), "l"(lo), "l"(hi) : "memory");
}
__device__ __forceinline__ double ll_pair_value(unsigned long long lo, unsigned long long hi) {
    return __longlong_as_double((long long)((hi << 32) | (lo & 0xFFFFFFFFull)));
}
__device__ __forceinline__ bool ll_pair_ok(unsigned long long lo, unsigned long long hi, unsigned tag) {
    return (unsigned)(lo >> 32) == tag && (unsigned)(hi >> 32) == tag;
}

template <bool SYS>
__device__ __forceinline__ void red_release_add_u64(unsigned long long* p, unsigned long long v) {
    if (SYS) asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
    else asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long gtimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// Peer waits give up after this long (a lost rank must not hang the GPU).
constexpr unsigned long long WATCHDOG_NS = 5000000000ull;

// fp32 parameter p -> fp64 smem replica
template <int MT>
__device__ __forceinline__ void put_param(TcSmem<MT>& S, int p, double v) {
    if (p < OFF_B0) {
        const int j = p / F;
        S.w0[j * SW0 + (p - j * F)] = v;
    } else if (p < OFF_W1) S.b0[p - OFF_B0] = v;
    else if (p < OFF_B1) {
        const int t = p - OFF_W1;
        S.w1[(t >> 6) * SW1 + (t & 63)] = v;
    } else if (p < OFF_W2) S.b1[p - OFF_B1] = v;
    else if (p < OFF_B2) S.w2[p - OFF_W2] = v;
    else S.b2[p - OFF_B2] = v;
}

template <int MT>
__device__ __forceinline__ double get_param(const TcSmem<MT>& S, int p) {
    if (p < OFF_B0) {
        const int j = p / F;
        return S.w0[j * SW0 + (p - j * F)];
    }
    if (p < OFF_W1) return S.b0[p - OFF_B0];
    if (p < OFF_B1) {
        const int t = p - OFF_W1;
        return S.w1[(t >> 6) * SW1 + (t & 63)];
    }
    if (p < OFF_W2) return S.b1[p - OFF_B1];
    if (p < OFF_B2) return S.w2[p - OFF_W2];
    return S.b2[p - OFF_B2];
}

template <int MT>
__device__ void load_params_plain(TcSmem<MT>& S, const float* __restrict__ p) {
    for (int t = threadIdx.x; t < NP / 2; t += NT) {
        const float2 v = __ldcg(reinterpret_cast<const float2*>(p) + t);
        put_param(S, 2 * t, (double)v.x);
        put_param(S, 2 * t + 1, (double)v.y);
    }
}

// All-gather of the LL words {tag, fp32 bits}: spin until every word this
// thread owns carries `tag`. False when the watchdog expired.
template <bool SYS, int MT>
__device__ bool load_params_ll(TcSmem<MT>& S, const unsigned long long* __restrict__ ll,
                               unsigned tag) {
    constexpr int PER = (NP + NT - 1) / NT;  // 10
    unsigned long long v[PER];
    unsigned pending = 0;
#pragma unroll
    for (int q = 0; q < PER; ++q)
        if (threadIdx.x + q * NT < NP) pending |= 1u << q;
    unsigned long long t0 = 0;
    for (unsigned it = 0; pending; ++it) {
#pragma unroll
        for (int q = 0; q < PER; ++q)
            if (pending & (1u << q)) v[q] = ld_relaxed_u64<SYS>(ll + threadIdx.x + q * NT);
#pragma unroll
        for (int q = 0; q < PER; ++q)
            if ((pending & (1u << q)) && (unsigned)(v[q] >> 32) == tag) pending &= ~(1u << q);
        if (pending && (it & 255) == 255) {
            const unsigned long long t = gtimer_ns();
            if (t0 == 0) t0 = t;
            else if (t - t0 > WATCHDOG_NS) return false;
        }
    }
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const int p = threadIdx.x + q * NT;
        if (p < NP) put_param(S, p, (double)__uint_as_float((unsigned)v[q]));
    }
    return true;
}

// Persistent per-thread gradient accumulators of one step.
struct TcGrads {
    double g1[2][2];  // gW1 tiles (mt = (w>>3) + 2q, nt = w & 7)
    double g0[3][2];  // [gW0|gb0]^T tiles (mt = (w>>3) + 2q over i, nt = w & 7 over j)
    double gx[2];     // warps 7..15: one extra tile (see tc_extra)
};

__device__ __forceinline__ void tc_zero(TcGrads& g) {
#pragma unroll
    for (int q = 0; q < 2; ++q) g.g1[q][0] = g.g1[q][1] = 0.0;
#pragma unroll
    for (int q = 0; q < 3; ++q) g.g0[q][0] = g.g0[q][1] = 0.0;
    g.gx[0] = g.gx[1] = 0.0;
}

// Extra K=TB tiles, one per warp 7..15: x = w - 7 in 0..3 is the G1 tile of
// m-tile x at n-tile 8 (column 64 of [H1|1] -> gb1); x in 4..8 is E n-tile x - 4.
constexpr int XW0 = 7;

// Visit every (parameter index, value) this thread accumulated.
template <typename Fn>
__device__ __forceinline__ void tc_for_each(const TcGrads& g, Fn fn) {
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int gq = lane >> 2, tq = lane & 3;
    const int nt = w & 7, mq = w >> 3;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const int k = (mq + 2 * q) * 8 + gq, j = nt * 8 + 2 * tq;
        fn(OFF_W1 + k * H1 + j, g.g1[q][0], g.g1[q][1], true);
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        const int i = (mq + 2 * q) * 8 + gq, j = nt * 8 + 2 * tq;
        if (i < F) {
            fn(OFF_W0 + j * F + i, g.g0[q][0], 0.0, false);
            fn(OFF_W0 + (j + 1) * F + i, g.g0[q][1], 0.0, false);
        } else if (i == F) {
            fn(OFF_B0 + j, g.g0[q][0], g.g0[q][1], true);
        }
    }
    const int x = w - XW0;
    if (x >= 0 && x < 4) {
        if (tq == 0) fn(OFF_B1 + x * 8 + gq, g.gx[0], 0.0, false);  // column 64
    } else if (x >= 4) {
        const int n = (x - 4) * 8 + 2 * tq;  // E column; row gq
        if (n < H2) {
            if (gq < A) fn(OFF_W2 + gq * H2 + n, g.gx[0], g.gx[1], true);
        } else if (n == H2) {
            if (gq < A) fn(OFF_B2 + gq, g.gx[0], 0.0, false);
            else if (gq == 2) fn(NP, g.gx[0], 0.0, false);
        }
    }
}

template <int MT>
__device__ void tc_prefetch(TcSmem<MT>& S, int buf, const TrainArgs& a, size_t r0, int nv) {
    constexpr int TB = 8 * MT;
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

// Ring prefetch (epoch kernel): record indices two tiles ahead, features and
// targets one tile ahead, gathered through the indices already in smem.
template <int MT>
__device__ __forceinline__ void tc_fetch_idx(TcSmem<MT>& S, int slot, const TrainArgs& a,
                                             uint32_t r0, int nv) {
    if ((int)threadIdx.x < nv) {
        const unsigned s = (unsigned)__cvta_generic_to_shared(&S.ord[slot][threadIdx.x]);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s),
                     "l"(a.order + r0 + threadIdx.x)
                     : "memory");
    }
}
template <int MT>
__device__ __forceinline__ void tc_fetch_rows(TcSmem<MT>& S, int slot, const TrainArgs& a, int nv) {
    constexpr int TB = 8 * MT;
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

// Constant columns: X col 44 = 1 (gb0), H1 col 64 = 1 (gb1), H2 col 32 = 1
// (gb2, KL), U cols 3.. = 0. Tiles never overwrite them.
template <int MT>
__device__ void tc_init_consts(TcSmem<MT>& S) {
    constexpr int TB = 8 * MT;
    for (int t = threadIdx.x; t < TB; t += NT) {
        for (int i = F; i < SX; ++i) S.x[t * SX + i] = i == F ? 1.0 : 0.0;
        for (int j = H1; j < SH1; ++j) S.h1[t * SH1 + j] = j == H1 ? 1.0 : 0.0;
        for (int k = H2; k < SH2; ++k) S.h2[t * SH2 + k] = k == H2 ? 1.0 : 0.0;
        for (int m = 0; m < SU; ++m) S.u[t * SU + m] = 0.0;
    }
}

// P0 of a tile, run ahead of it (overlapping the previous step's
// synchronisation): staged fp32 rows -> fp64 X (cols 0..43) and the clamped
// log-targets ln(t^_a) the KL term needs. Caller: cp.async complete + barrier
// before, barrier after.
template <int MT>
__device__ void tc_stage_in(TcSmem<MT>& S, int slot, int loss_mode, int t0 = 0) {
    constexpr int TB = 8 * MT;
    const int tid = threadIdx.x;
    for (int t = tid - t0; t < TB * F; t += NT - t0) {
        const int r = t / F;
        S.x[r * SX + (t - r * F)] = (double)S.stage_f[slot][t];
    }
    if (tid >= NT - 2 * TB) {
        const int q = tid - (NT - 2 * TB);
        // KL: ln(clamp(target)); TD: the raw (action, reward) record
        S.ltgt[q] = loss_mode == 1 ? S.stage_t[slot][q] : log(clampp(S.stage_t[slot][q]));
    }
}

__device__ __forceinline__ void pair_sync(int id) {
    asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory");
}

// One tile of 8*MT records (rows >= nv are zero padding and contribute 0);
// X and ltgt already staged by tc_stage_in.
//
// Record chain, per m-tile, on a warp pair (warps 2p, 2p+1 own m-tile p; they
// synchronise with a 64-thread named barrier only, so pairs drift freely and
// one pair's softmax overlaps the others' tensor work):
//   F1 (n-tiles 4h..4h+3) | F2 (n-tiles 2h, 2h+1) | F3 + B1 | B2 (n-tiles 4h..4h+3)
// then one CTA barrier and the gradient phase over all records (all warps):
//   G1 (+ gb1 via H1's ones column), E, G0 (+ gb0 via X's ones column).
template <int MT, bool VAR>
__device__ void tc_tile(TcSmem<MT>& S, TcGrads& g, int nv, double inv_b, int loss_mode) {
    constexpr int TB = 8 * MT;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int gq = lane >> 2, tq = lane & 3;

    if (w < 2 * MT) {
        const int p = w >> 1, h = w & 1, bar = 1 + p;
        const int r = p * 8 + gq;  // this lane's record row in A fragments / C rows
        // ---- F1: H1[p-tile][n-tiles 4h..4h+3] = relu(X W0^T + b0), K = 44
        {
            double acc[4][2];
#pragma unroll
            for (int nn = 0; nn < 4; ++nn) {
                const int c = (4 * h + nn) * 8 + 2 * tq;
                acc[nn][0] = S.b0[c];
                acc[nn][1] = S.b0[c + 1];
            }
            const double* xa = S.x + r * SX + tq;
            const double* wb = S.w0 + ((4 * h) * 8 + gq) * SW0 + tq;
#pragma unroll
            for (int k0 = 0; k0 < F; k0 += 4) {
                const double af = xa[k0];
#pragma unroll
                for (int nn = 0; nn < 4; ++nn) dmma(acc[nn], af, wb[nn * 8 * SW0 + k0]);
            }
#pragma unroll
            for (int nn = 0; nn < 4; ++nn) {
                double* o = S.h1 + r * SH1 + (4 * h + nn) * 8 + 2 * tq;
                o[0] = acc[nn][0] > 0.0 ? acc[nn][0] : 0.0;
                o[1] = acc[nn][1] > 0.0 ? acc[nn][1] : 0.0;
            }
        }
        pair_sync(bar);
        TC_MARK(1);
        // ---- F2: H2[p-tile][n-tiles 2h, 2h+1] = relu(H1 W1^T + b1), K = 64
        {
            double acc[2][2];
#pragma unroll
            for (int nn = 0; nn < 2; ++nn) {
                const int c = (2 * h + nn) * 8 + 2 * tq;
                acc[nn][0] = S.b1[c];
                acc[nn][1] = S.b1[c + 1];
            }
            const double* ha = S.h1 + r * SH1 + tq;
            const double* wb = S.w1 + ((2 * h) * 8 + gq) * SW1 + tq;
#pragma unroll
            for (int k0 = 0; k0 < H1; k0 += 4) {
                const double af = ha[k0];
#pragma unroll
                for (int nn = 0; nn < 2; ++nn) dmma(acc[nn], af, wb[nn * 8 * SW1 + k0]);
            }
#pragma unroll
            for (int nn = 0; nn < 2; ++nn) {
                double* o = S.h2 + r * SH2 + (2 * h + nn) * 8 + 2 * tq;
                o[0] = acc[nn][0] > 0.0 ? acc[nn][0] : 0.0;
                o[1] = acc[nn][1] > 0.0 ? acc[nn][1] : 0.0;
            }
        }
        pair_sync(bar);
        TC_MARK(2);
        // ---- F3 + B1 on the pair's first warp (the FP64 softmax is the only
        //      work here; the partner waits at the pair barrier instead of
        //      duplicating it on the shared FP64 pipe)
        if (h == 0) {
            // two independent accumulator chains (even / odd k-steps), summed
            double lg[2], lh[2] = {0.0, 0.0};
            lg[0] = tq == 0 ? S.b2[0] : 0.0;
            lg[1] = tq == 0 ? S.b2[1] : 0.0;
            const double* hb = S.h2 + r * SH2 + tq;
#pragma unroll
            for (int k0 = 0; k0 < H2; k0 += 8) {
                dmma(lg, hb[k0], gq < A ? S.w2[gq * H2 + k0 + tq] : 0.0);
                dmma(lh, hb[k0 + 4], gq < A ? S.w2[gq * H2 + k0 + 4 + tq] : 0.0);
            }
            lg[0] += lh[0];
            lg[1] += lh[1];
            TC_MARK(11);
            const double l0 = __shfl_sync(0xffffffffu, lg[0], lane & ~3);
            const double l1 = __shfl_sync(0xffffffffu, lg[1], lane & ~3);
            const int a = tq & 1;
            const bool valid = r < nv;
            double loss, d3;
            if (VAR && loss_mode == 1) {
                // TD / reward regression: Q = the raw outputs, record (act, reward)
                const int act = S.ltgt[2 * r] != 0.0 ? 1 : 0;
                const double err = (act ? l1 : l0) - S.ltgt[2 * r + 1];
                loss = err * err;
                d3 = (valid && tq == act) ? 2.0 * err * inv_b : 0.0;
            } else {
                // log-softmax form: with d = l_a - l_other, z = exp(-|d|),
                //   p_a = (d >= 0 ? 1 : z) / (1 + z),  ln p_a = min(d, 0) - log1p(z)
                // (equal to the reference's exp / sum / log(p/t) up to fp64 rounding)
                const double d = a ? l1 - l0 : l0 - l1;
                const double z = exp(-fabs(d));
                const double lse = log1p(z);
                // 1 / (1 + z), 1 <= 1 + z <= 2: hardware reciprocal + Newton steps
                const double den = 1.0 + z;
                double rc;
                asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rc) : "d"(den));
                rc = fma(rc, fma(-den, rc, 1.0), rc);
                rc = fma(rc, fma(-den, rc, 1.0), rc);
                rc = fma(rc, fma(-den, rc, 1.0), rc);
                const double pa = d >= 0.0 ? rc : z * rc;
                const double lpc = pa < 1e-7 ? LN_PMIN : (pa > 1.0 - 1e-7 ? LN_PMAX : fmin(d, 0.0) - lse);
                const double pc = clampp(pa);
                const double lr = lpc - S.ltgt[2 * r + a];
                const double term = pc * lr;
                const double to = __shfl_xor_sync(0xffffffffu, term, 1);
                loss = a ? to + term : term + to;
                d3 = (valid && tq < 2) ? pa * (lr - loss) * inv_b : 0.0;
            }
            TC_MARK(12);
            if (tq < 2) S.u[r * SU + tq] = d3;
            if (tq == 0) S.u[r * SU + 2] = valid ? loss : 0.0;
#pragma unroll
            for (int nt = 0; nt < H2 / 8; ++nt) {
                double dd[2] = {0.0, 0.0};
                dmma(dd, d3, tq < A ? S.w2[tq * H2 + nt * 8 + gq] : 0.0);
                const int k = nt * 8 + 2 * tq;
                const double* hh = S.h2 + r * SH2 + k;
                S.d2[r * SH2 + k] = hh[0] <= 0.0 ? 0.0 : dd[0];
                S.d2[r * SH2 + k + 1] = hh[1] <= 0.0 ? 0.0 : dd[1];
            }
        }
        pair_sync(bar);
        TC_MARK(3);
        // ---- B2: D1[p-tile][n-tiles 4h..4h+3] = (D2 W1) o [h1 > 0], K = 32
        {
            double acc[4][2];
#pragma unroll
            for (int nn = 0; nn < 4; ++nn) acc[nn][0] = acc[nn][1] = 0.0;
            const double* da = S.d2 + r * SH2 + tq;
            const double* wb = S.w1 + tq * SW1 + (4 * h) * 8 + gq;  // B[k][j] = W1[k][j]
#pragma unroll
            for (int k0 = 0; k0 < H2; k0 += 4) {
                const double af = da[k0];
#pragma unroll
                for (int nn = 0; nn < 4; ++nn) dmma(acc[nn], af, wb[k0 * SW1 + nn * 8]);
            }
#pragma unroll
            for (int nn = 0; nn < 4; ++nn) {
                const int j = (4 * h + nn) * 8 + 2 * tq;
                S.d1[r * SH1 + j] = S.h1[r * SH1 + j] <= 0.0 ? 0.0 : acc[nn][0];
                S.d1[r * SH1 + j + 1] = S.h1[r * SH1 + j + 1] <= 0.0 ? 0.0 : acc[nn][1];
            }
        }
    }
    __syncthreads();
    TC_MARK(4);

    // ---- gradient phase, K = records of the tile (accumulators persist over the step)
    {
        const int nt = w & 7, mq = w >> 3;
        // G1: A[k][r] = D2[r][k], B[r][j] = H1[r][j]; m-tiles (k) mq + 2q, n-tile nt
        {
            const double* ab = S.d2 + tq * SH2 + mq * 8 + gq;
            const double* bb = S.h1 + tq * SH1 + nt * 8 + gq;
#pragma unroll
            for (int r0 = 0; r0 < TB; r0 += 4) {
                const double bf = bb[r0 * SH1];
                dmma(g.g1[0], ab[r0 * SH2], bf);
                dmma(g.g1[1], ab[r0 * SH2 + 16], bf);
            }
        }
        const int x = w - XW0;
        if (x >= 0) {
            // x < 4: A = D2^T (m-tile x), B = H1 cols 64..71; x >= 4: A = U^T, B = H2 cols 8(x-4)..
            const double* xa = x < 4 ? S.d2 + tq * SH2 + x * 8 + gq : S.u + tq * SU + gq;
            const int sa = x < 4 ? SH2 : SU;
            const double* xb = x < 4 ? S.h1 + tq * SH1 + H1 + gq : S.h2 + tq * SH2 + (x - 4) * 8 + gq;
            const int sb = x < 4 ? SH1 : SH2;
#pragma unroll 7
            for (int r0 = 0; r0 < TB; r0 += 4) dmma(g.gx, xa[r0 * sa], xb[r0 * sb]);
        }
        // G0: [gW0|gb0]^T += [X|1]^T D1: A[i][r] = X[r][i], B[r][j] = D1[r][j]
        {
            const double* ab = S.x + tq * SX + mq * 8 + gq;
            const double* bb = S.d1 + tq * SH1 + nt * 8 + gq;
#pragma unroll 2
            for (int r0 = 0; r0 < TB; r0 += 4) {
                const double bf = bb[r0 * SH1];
                const double* ar = ab + r0 * SX;
                dmma(g.g0[0], ar[0], bf);
                dmma(g.g0[1], ar[16], bf);
                dmma(g.g0[2], ar[32], bf);
            }
        }
    }
    TC_MARK(5);
    // (the caller's next __syncthreads orders the gradient reads of X / D1 / H1
    //  before the next tile overwrites them)
}

// Per-step record slice of CTA `cta` (rank-major, then CTA-major; identical to
// k_train.cu's step_slice).
__device__ __forceinline__ void tc_slice(const TrainArgs& a, int rank, int nranks, long step,
                                         int cta, int nctas, uint32_t& lo, uint32_t& hi,
                                         uint32_t& nb) {
    const uint32_t n = (uint32_t)a.n, batch = (uint32_t)a.batch;
    const uint32_t start = (uint32_t)step * batch;
    const uint32_t stop = min(n, start + batch);
    nb = stop - start;
    const uint32_t per_rank = (nb + nranks - 1) / (uint32_t)nranks;
    const uint32_t r_lo = min(stop, start + (uint32_t)rank * per_rank);
    const uint32_t r_hi = min(stop, r_lo + per_rank);
    const uint32_t per_cta = (r_hi - r_lo + nctas - 1) / (uint32_t)nctas;
    lo = min(r_hi, r_lo + (uint32_t)cta * per_cta);
    hi = min(r_hi, lo + per_cta);
}

// This CTA's slice of a FULL step is the same at every step up to the offset
// step * batch: computed once per launch (two integer divisions per call
// otherwise, ~4 calls per step on every thread); only a final partial step
// takes the general path.
struct TcWho {
    int rank, nranks, cta, nctas;
    uint32_t lo_off, hi_off;  // slice of a full step, relative to its start
};

__device__ __forceinline__ TcWho tc_who(const TrainArgs& a, int rank, int nranks, int cta,
                                        int nctas) {
    TcWho w{rank, nranks, cta, nctas, 0u, 0u};
    const uint32_t batch = (uint32_t)a.batch;
    const uint32_t per_rank = (batch + nranks - 1) / (uint32_t)nranks;
    const uint32_t r_lo = min(batch, (uint32_t)rank * per_rank);
    const uint32_t r_hi = min(batch, r_lo + per_rank);
    const uint32_t per_cta = (r_hi - r_lo + nctas - 1) / (uint32_t)nctas;
    w.lo_off = min(r_hi, r_lo + (uint32_t)cta * per_cta);
    w.hi_off = min(r_hi, w.lo_off + per_cta);
    return w;
}

__device__ __forceinline__ void tc_slice_w(const TrainArgs& a, const TcWho& w, long step,
                                           uint32_t& lo, uint32_t& hi, uint32_t& nb) {
    const uint32_t batch = (uint32_t)a.batch, start = (uint32_t)step * batch;
    if ((size_t)start + batch <= a.n) {
        lo = start + w.lo_off;
        hi = start + w.hi_off;
        nb = batch;
    } else {
        tc_slice(a, w.rank, w.nranks, step, w.cta, w.nctas, lo, hi, nb);
    }
}

// Next tile after (step, r0) within [step, n_steps); r0 == UINT32_MAX asks for
// the first tile of `step`.
template <int TB>
__device__ bool tc_next(const TrainArgs& a, const TcWho& who, long n_steps, long& step,
                        uint32_t& r0, int& nv) {
    uint32_t lo, hi, nb;
    if (r0 != 0xFFFFFFFFu) {
        tc_slice_w(a, who, step, lo, hi, nb);
        if (r0 + TB < hi) {
            r0 += TB;
            nv = (int)min((uint32_t)TB, hi - r0);
            return true;
        }
        ++step;
    }
    for (; step < n_steps; ++step) {
        tc_slice_w(a, who, step, lo, hi, nb);
        if (hi > lo) {
            r0 = lo;
            nv = (int)min((uint32_t)TB, hi - lo);
            return true;
        }
    }
    return false;
}

// Stores this thread's accumulators into partial row `part` (parameter order,
// loss at NP).
__device__ __forceinline__ void tc_store_partial(const TcGrads& g, double* __restrict__ part) {
    tc_for_each(g, [&](int p, double v0, double v1, bool pair) {
        if (pair) __stcg(reinterpret_cast<double2*>(part + p), make_double2(v0, v1));
        else __stcg(part + p, v0);
    });
}

// Final owner of parameter p: SGD w = float(double(w) - lr * g)
// (policy.cpp:328-332) or Adam, published as {tag, fp32 bits} to every rank.
template <bool SYS, int MT, bool VAR>
__device__ __forceinline__ void tc_update_publish(TcSmem<MT>& S, const TrainArgs& a, int p, double gsum,
                                                  unsigned tag, int R, bool adam_smem, int own_lo,
                                                  double adam_c1, double adam_c2) {
    double upd;
    if (VAR && a.optimizer == 1) {
        // Adam: this CTA owns the moments of its slice across steps — in
        // shared memory for the epoch when the slice fits (no global round
        // trip on the step's critical path)
        double* pm = adam_smem ? &S.adam[0][p - own_lo] : &a.adam_m[p];
        double* pv = adam_smem ? &S.adam[1][p - own_lo] : &a.adam_v[p];
        const double m = a.beta1 * *pm + (1.0 - a.beta1) * gsum;
        const double v = a.beta2 * *pv + (1.0 - a.beta2) * gsum * gsum;
        *pm = m;
        *pv = v;
        upd = a.lr * (m / adam_c1) / (sqrt(v / adam_c2) + a.adam_eps);
    } else {
        upd = a.lr * gsum;
    }
    const float nw = __double2float_rn(get_param(S, p) - upd);
    const unsigned long long word = ((unsigned long long)tag << 32) | __float_as_uint(nw);
    for (int r = 0; r < R; ++r) st_relaxed_u64<SYS>(a.llp[r] + p, word);
}

}  // namespace

size_t train_tc_smem_bytes(int mt) { return mt == 4 ? sizeof(TcSmem<4>) : sizeof(TcSmem<7>); }

template <int MT, bool SYS, bool VAR>
__global__ void __launch_bounds__(NT, 1) train_epoch_tc_kernel(TrainArgs a) {
    constexpr int TB = 8 * MT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TcSmem<MT>& S = *reinterpret_cast<TcSmem<MT>*>(smem_raw);
    if (*a.diverged_epoch >= 0 || *a.status != 0) return;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    // peer set: R ranks x Gl CTAs; this CTA is (rank, c), global index gc
    const int R = a.peers;
    const int Gl = a.pvirt ? (int)gridDim.x / R : (int)gridDim.x;
    const int rank = a.pvirt ? (int)blockIdx.x / Gl : a.prank;
    const int c = a.pvirt ? (int)blockIdx.x % Gl : (int)blockIdx.x;
    const int GG = R * Gl, gc = rank * Gl + c;
    const TcWho who = tc_who(a, rank, R, c, Gl);
    const long n_steps = (long)((a.n + a.batch - 1) / a.batch);
    // Two-level reduce-scatter, balanced splits (every slice non-empty):
    //   level 1 (within a rank): CTA c sums element 0 = the loss and params
    //     [p_lo, p_hi) (a 1/Gl slice) over its own rank's Gl partial rows — with
    //     one rank that sum is final;
    //   level 2 (peer sets, R > 1): CTA gc sums the loss and params [q_lo, q_hi)
    //     (a 1/GG slice) over the R per-GPU sums, read as LL pairs over NVLink
    //     (R x 5,027 pairs cross the fabric per step, not R x Gl partial rows).
    // Every CTA owns parameters at the final level, so every CTA publishes LL
    // words after its reads of the step's rows: no CTA can overwrite its row
    // (next step) before all reads of it are done.
    const int p_lo = (int)(((long)c * NP) / Gl), p_hi = (int)(((long)(c + 1) * NP) / Gl);
    const int q_lo = (int)(((long)gc * NP) / GG), q_hi = (int)(((long)(gc + 1) * NP) / GG);
    const int own_lo = R == 1 ? p_lo : q_lo, own_hi = R == 1 ? p_hi : q_hi;
    const int n_elem = 1 + (p_hi - p_lo);
    // reduction layout: EB elements x SUB source subsets (EB * SUB = NT)
    int EB = 8;
    while (EB < 64 && EB < n_elem) EB <<= 1;
    const int SUB = NT / EB;
    double* my_part = a.part[rank] + (size_t)c * PSTR;
    unsigned long long* my_ctr = a.ctr[rank];
    const unsigned long long* my_llp = a.llp[rank];
    bool aborted = false, diverged_here = false;

    // Pipeline (tile k): rows of tile k+1 and indices of tile k+2 are fetched
    // (cp.async) at the top of tile k; tile k+1 is staged into X (P0) right
    // after tile k, overlapping the step synchronisation.
    // Cursors: c1 = tile k+1, c2 = tile k+2.
    long s1 = 0, s2 = 0;
    uint32_t r1 = 0xFFFFFFFFu, r2;
    int n1 = 0, n2 = 0;
    bool h1 = tc_next<TB>(a, who, n_steps, s1, r1, n1);  // tile 0
    if (h1) tc_fetch_idx(S, 0, a, r1, n1);
    s2 = s1; r2 = r1;
    bool h2 = h1 && tc_next<TB>(a, who, n_steps, s2, r2, n2);  // tile 1
    if (h2) tc_fetch_idx(S, 1, a, r2, n2);
    cp_async_commit();
    // Adam moments of the slice on chip for the whole epoch (written back at
    // the end of the launch); a lone CTA or a slice wider than 64 keeps them
    // in global memory
    const bool adam_smem = VAR && a.optimizer == 1 && GG > 1 && own_hi - own_lo <= 64;
    if (adam_smem && tid < own_hi - own_lo) {
        S.adam[0][tid] = a.adam_m[own_lo + tid];
        S.adam[1][tid] = a.adam_v[own_lo + tid];
    }
    load_params_plain(S, a.params);
    tc_init_consts(S);
    cp_async_wait_all();
    __syncthreads();
    if (h1) tc_fetch_rows(S, 0, a, n1);  // tile 0 rows
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
    if (h1) tc_stage_in(S, 0, a.loss_mode);
    // shift: c1 <- tile 1, c2 <- tile 2
    h1 = h2; s1 = s2; r1 = r2; n1 = n2;
    s2 = s1; r2 = r1;
    h2 = h1 && tc_next<TB>(a, who, n_steps, s2, r2, n2);
    TcGrads g;
    tc_zero(g);
    double epoch_total = 0.0;
    int k = 0;  // tile counter: tile k's rows in stage[k & 1], its indices were in ord[k & 1]
    bool stage_due = false;  // tile k (next to compute) fetched but not yet staged into X
    TC_MARK(-1);

    for (long step = 0; step < n_steps; ++step) {
        uint32_t lo, hi, nb;
        tc_slice_w(a, who, step, lo, hi, nb);
        const double inv_b = 1.0 / (double)nb;
        const unsigned tag = a.tag_base + (unsigned)step + 1u;
        // Adam's bias corrections for this step, computed up front (two pow()s
        // off the critical path between the slice reduce and the publish)
        double adam_c1 = 1.0, adam_c2 = 1.0;
        if (VAR && a.optimizer == 1 && tid < (R == 1 ? 64 : NT / R)) {
            const double t = (double)(a.step0 + (unsigned)step + 1u);
            adam_c1 = 1.0 - pow(a.beta1, t);
            adam_c2 = 1.0 - pow(a.beta2, t);
        }
        TC_TRACE(step, 0);
        for (uint32_t r0 = lo; r0 < hi; r0 += TB, ++k) {
            const int nv = (int)min((uint32_t)TB, hi - r0);
            __syncthreads();  // tile k staged; replicas (re)loaded
            const bool more = h1;
            if (h1) tc_fetch_rows(S, (k + 1) & 1, a, n1);     // rows of tile k+1
            if (h2) tc_fetch_idx(S, k & 1, a, r2, n2);        // indices of tile k+2
            cp_async_commit();
            h1 = h2; s1 = s2; r1 = r2; n1 = n2;
            if (h2) h2 = tc_next<TB>(a, who, n_steps, s2, r2, n2);
            TC_MARK(6);
            tc_tile<MT, VAR>(S, g, nv, inv_b, a.loss_mode);
            if (more && r0 + TB < hi) {
                // the next tile belongs to this step: stage it now
                cp_async_wait_all();
                __syncthreads();
                tc_stage_in(S, (k + 1) & 1, a.loss_mode);
                TC_MARK(0);
            } else {
                stage_due = more;  // staged after this step's partial is published
            }
        }
        // (only the variant instantiations ever run a lone CTA: the
        //  reference's KL + SGD uses the bit-exact 1-CTA kernel there)
        if (VAR && GG == 1) {
            // ---- a lone CTA (small batches, e.g. the variants at B <= 32):
            //      its partial IS the batch gradient, so the update is applied
            //      in place — no partial rows, counter or LL words
            tc_for_each(g, [&](int p, double v0, double, bool) {
                if (p == NP) {
                    const double loss = v0 / (double)nb;
                    S.scal[0] = loss;
                    S.scal[1] = isfinite(loss) ? 0.0 : 1.0;
                }
            });
            if (stage_due) cp_async_wait_all();
            __syncthreads();
            if (S.scal[1] != 0.0) {
                if (tid == 0) *a.diverged_epoch = a.epoch;
                diverged_here = true;
                break;
            }
            if (tid == 0) epoch_total = fma(S.scal[0], (double)nb, epoch_total);
            const bool adam = VAR && a.optimizer == 1;
            double c1 = 1.0, c2 = 1.0;
            if (adam) {
                const double t_adam = (double)(a.step0 + (unsigned)step + 1u);
                c1 = 1.0 - pow(a.beta1, t_adam);
                c2 = 1.0 - pow(a.beta2, t_adam);
            }
            auto apply = [&](int p, double gsum) {
                double upd;
                if (adam) {
                    const double m = a.beta1 * a.adam_m[p] + (1.0 - a.beta1) * gsum;
                    const double v = a.beta2 * a.adam_v[p] + (1.0 - a.beta2) * gsum * gsum;
                    a.adam_m[p] = m;
                    a.adam_v[p] = v;
                    upd = a.lr * (m / c1) / (sqrt(v / c2) + a.adam_eps);
                } else {
                    upd = a.lr * gsum;
                }
                put_param(S, p, (double)__double2float_rn(get_param(S, p) - upd));
            };
            tc_for_each(g, [&](int p, double v0, double v1, bool pair) {
                if (p >= NP) return;
                apply(p, v0);
                if (pair) apply(p + 1, v1);
            });
            tc_zero(g);
            if (stage_due) {
                __syncthreads();
                tc_stage_in(S, k & 1, a.loss_mode);
            }
            stage_due = false;
            continue;  // the loop top's barrier publishes the replicas
        }
        // ---- 1. publish this CTA's partial
        tc_store_partial(g, my_part);
        if (stage_due) cp_async_wait_all();  // this thread's copies of the next tile
        __syncthreads();                      // partial issued, gradient phase done, rows landed
        // ---- 2. arrive on this rank's counter (rows and counter are local to
        //      the GPU: GPU scope even in a peer set); wait (warp 0) until all
        //      Gl CTAs of the rank arrived while warps 1..15 stage the next tile
        if (tid == 0) {
            red_release_add_u64<false>(my_ctr, 1ull);
            TC_MARK(7);
            TC_TRACE(step, 1);
            const unsigned long long target =
                a.ctr_base + (unsigned long long)(step + 1) * (unsigned long long)Gl;
            unsigned long long t0 = 0;
            for (unsigned it = 0; ld_acquire_u64<false>(my_ctr) < target; ++it) {
                if ((it & 255) == 255) {
                    const unsigned long long t = gtimer_ns();
                    if (t0 == 0) t0 = t;
                    else if (t - t0 > WATCHDOG_NS) {
                        S.scal[1] = 2.0;  // abort
                        break;
                    }
                }
            }
        } else if (stage_due && tid >= 32) {
            tc_stage_in(S, k & 1, a.loss_mode, 32);
        }
        stage_due = false;
        __syncthreads();
        TC_MARK(8);
        TC_TRACE(step, 2);
        if (S.scal[1] == 2.0) {
            aborted = true;
            break;
        }
        // ---- 3. level 1: reduce [loss | slice] over this rank's Gl partial
        //      rows, fixed association: thread (e, s) folds rows s, s + SUB, ...
        //      (all loads in flight at once: one L2 round trip), then thread e
        //      sums the SUB subset totals in order
        bool diverged = false;
        for (int e0 = 0; e0 < n_elem; e0 += EB) {
            const int e = e0 + tid % EB, sb = tid / EB;
            double v = 0.0;
            if (e < n_elem) {
                const int p = e == 0 ? NP : p_lo + e - 1;
                const double* src = a.part[rank] + p;
                double u[20];
#pragma unroll
                for (int j = 0; j < 20; ++j) {
                    const int q = sb + j * SUB;
                    u[j] = q < Gl ? __ldcg(src + (size_t)q * PSTR) : 0.0;
                }
#pragma unroll
                for (int j = 0; j < 20; ++j) v += u[j];
                for (int q = sb + 20 * SUB; q < Gl; q += SUB) v += __ldcg(src + (size_t)q * PSTR);
            }
            S.red[sb * EB + tid % EB] = v;
            __syncthreads();
            if (tid < EB) {
                double t = 0.0;
                for (int q = 0; q < SUB; ++q) t += S.red[q * EB + tid];
                S.red[NT + tid] = t;
                if (e0 == 0 && tid == 0) {
                    const double loss = t / (double)nb;
                    S.scal[0] = loss;
                    S.scal[1] = (R > 1 || isfinite(loss)) ? 0.0 : 1.0;  // peer sets: level 2 decides
                }
            }
            __syncthreads();
            if (S.scal[1] != 0.0) {
                diverged = true;
                break;
            }
            // ---- 4. one rank: SGD on the slice, {tag, fp32} words to the
            //      rank; peer set: the per-GPU sum as an LL pair (the loss by c 0)
            if (tid < EB) {
                const int e2 = e0 + tid;
                if (e2 < n_elem && R > 1) {
                    if (e2 >= 1) st_ll_pair<SYS>(a.gp[rank] + 2 * (size_t)(p_lo + e2 - 1), S.red[NT + tid], tag);
                    else if (c == 0) st_ll_pair<SYS>(a.gp[rank] + 2 * (size_t)NP, S.red[NT + tid], tag);
                } else if (e2 >= 1 && e2 < n_elem) {
                    tc_update_publish<SYS, MT, VAR>(S, a, p_lo + e2 - 1, S.red[NT + tid], tag, R, adam_smem,
                                                     own_lo, adam_c1, adam_c2);
                }
            }
            __syncthreads();  // S.red reuse
        }
        // ---- 5. level 2 (peer sets): thread (e, r) reads rank r's per-GPU
        //      sum of element e (0 = loss, then params [q_lo, q_hi)) over
        //      NVLink; thread e sums them in rank order -> identical values on
        //      every rank; the loss decides divergence before any publish
        if (R > 1 && !diverged) {
            const int n2 = 1 + (q_hi - q_lo), per = NT / R;
            for (int e0 = 0; e0 < n2; e0 += per) {
                const int e = e0 + tid / R, r = tid % R;
                if (tid < per * R && e < n2) {
                    const unsigned long long* src = a.gp[r] + 2 * (size_t)(e == 0 ? NP : q_lo + e - 1);
                    unsigned long long lo = 0, hi = 0;
                    unsigned long long t0 = 0;
                    for (unsigned it = 0;; ++it) {
                        ld_v2<SYS>(src, lo, hi);
                        if (ll_pair_ok(lo, hi, tag)) break;
                        if ((it & 255) == 255) {
                            const unsigned long long t = gtimer_ns();
                            if (t0 == 0) t0 = t;
                            else if (t - t0 > WATCHDOG_NS) {
                                S.scal[1] = 2.0;
                                break;
                            }
                        }
                    }
                    S.red[tid] = ll_pair_value(lo, hi);
                }
                __syncthreads();
                if (S.scal[1] == 2.0) break;
                if (tid < per && e0 + tid < n2) {
                    double t = 0.0;
                    for (int q = 0; q < R; ++q) t += S.red[tid * R + q];
                    if (e0 + tid == 0) {
                        const double loss = t / (double)nb;
                        S.scal[0] = loss;
                        S.scal[1] = isfinite(loss) ? 0.0 : 1.0;
                    }
                    S.red[NT + tid] = t;
                }
                __syncthreads();
                if (S.scal[1] != 0.0) {
                    diverged = S.scal[1] == 1.0;
                    break;
                }
                if (tid < per && e0 + tid >= 1 && e0 + tid < n2)
                    tc_update_publish<SYS, MT, VAR>(S, a, q_lo + e0 + tid - 1, S.red[NT + tid], tag, R,
                                                     adam_smem, own_lo, adam_c1, adam_c2);
                __syncthreads();  // S.red reuse
            }
            if (S.scal[1] == 2.0) {
                aborted = true;
                break;
            }
        }
        if (diverged) {
            if (c == 0 && tid == 0) *a.diverged_epoch = a.epoch;
            diverged_here = true;
            break;
        }
        TC_MARK(9);
        TC_TRACE(step, 3);
        if (tid == 0) epoch_total = fma(S.scal[0], (double)nb, epoch_total);
        // ---- 5. all-gather the new parameters into the fp64 replicas
        if (!load_params_ll<SYS>(S, my_llp, tag)) S.scal[1] = 2.0;
        tc_zero(g);
        __syncthreads();
        if (S.scal[1] == 2.0) {
            aborted = true;
            break;
        }
        TC_MARK(10);
        TC_TRACE(step, 4);
    }
    cp_async_wait_all();
    __syncthreads();  // a lone CTA's last in-place update is visible to every thread
    if (aborted) {
        if (tid == 0) atomicExch(a.status, 1);
        return;
    }
    if (adam_smem && tid < own_hi - own_lo) {  // the slice's moments for the next epoch
        a.adam_m[own_lo + tid] = S.adam[0][tid];
        a.adam_v[own_lo + tid] = S.adam[1][tid];
    }
    // rank-local outputs: params (fp32 values of the replicas) and the epoch loss.
    // On divergence the replicas hold the parameters after the last finite
    // step (the loop leaves before that step's words are gathered), which is
    // what the reference's net holds when fit throws (policy.cpp:321-325).
    if (c == 0 && (!a.pvirt || rank == 0)) {
        for (int t = tid; t < NP; t += NT) a.params[t] = (float)get_param(S, t);
        if (tid == 0 && !diverged_here) a.epoch_loss[a.epoch] = epoch_total / (double)a.n;
    }
}

// Data-parallel path: one step's per-CTA partials (the reduction, NCCL
// all-reduce and SGD update follow as separate launches).
template <int MT>
__global__ void __launch_bounds__(NT, 1) train_partial_tc_kernel(TrainArgs a, long step) {
    constexpr int TB = 8 * MT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TcSmem<MT>& S = *reinterpret_cast<TcSmem<MT>*>(smem_raw);
    if (*a.diverged_epoch >= 0) return;
    uint32_t lo, hi, nb;
    tc_slice(a, a.rank, a.nranks, step, blockIdx.x, gridDim.x, lo, hi, nb);
    if (hi > lo) tc_prefetch<MT>(S, 0, a, lo, (int)min((uint32_t)TB, hi - lo));
    load_params_plain(S, a.params);
    tc_init_consts(S);
    TcGrads g;
    tc_zero(g);
    const double inv_b = 1.0 / (double)nb;
    int buf = 0;
    for (uint32_t r0 = lo; r0 < hi; r0 += TB) {
        const int nv = (int)min((uint32_t)TB, hi - r0);
        cp_async_wait_all();
        __syncthreads();
        tc_stage_in(S, buf, a.loss_mode);
        __syncthreads();
        buf ^= 1;
        if (r0 + TB < hi) tc_prefetch<MT>(S, buf, a, r0 + TB, (int)min((uint32_t)TB, hi - r0 - TB));
        tc_tile<MT, false>(S, g, nv, inv_b, 0);
    }
    tc_store_partial(g, a.partials + (size_t)blockIdx.x * PSTR);
}

template __global__ void train_epoch_tc_kernel<4, false, false>(TrainArgs);
template __global__ void train_epoch_tc_kernel<7, false, false>(TrainArgs);
template __global__ void train_epoch_tc_kernel<4, true, false>(TrainArgs);
template __global__ void train_epoch_tc_kernel<7, true, false>(TrainArgs);
template __global__ void train_epoch_tc_kernel<4, false, true>(TrainArgs);
template __global__ void train_epoch_tc_kernel<7, false, true>(TrainArgs);
template __global__ void train_epoch_tc_kernel<4, true, true>(TrainArgs);
template __global__ void train_epoch_tc_kernel<7, true, true>(TrainArgs);
template __global__ void train_partial_tc_kernel<4>(TrainArgs, long);
template __global__ void train_partial_tc_kernel<7>(TrainArgs, long);

}  // namespace gbxcu

#ifdef GBX_PHASE_TIMING
extern "C" int gbxcu_debug_phase_cycles_tc(unsigned long long* out, int reset) {
    if (cudaMemcpyFromSymbol(out, gbxcu::g_tc_phase, sizeof(unsigned long long) * 16) != cudaSuccess)
        return 3;
    if (reset) {
        unsigned long long z[16] = {};
        cudaMemcpyToSymbol(gbxcu::g_tc_phase, z, sizeof(z));
    }
    return 0;
}
extern "C" int gbxcu_debug_trace_tc(unsigned long long* out) {
    return cudaMemcpyFromSymbol(out, gbxcu::g_tc_trace, sizeof(unsigned long long) * 8 * 160 * 6) ==
                   cudaSuccess ? 0 : 3;
}
#endif
