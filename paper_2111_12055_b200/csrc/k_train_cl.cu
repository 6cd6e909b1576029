// k_train_cl.cu — the bit-exact batch-32 train epoch (the reference's default
// TrainConfig::batch_size) on a 4-CTA thread-block cluster, sm_100a.
//
// Replaces fit's inner loop (proj/src/policy.cpp:316-333) like
// train_epoch_kernel<32> (k_train.cu) with the same arithmetic, in the same
// order: every forward / backward output and every parameter's gradient is a
// sequential chain owned by ONE thread, exactly the reference's summation
// order (F1 DFMA — fp32 x fp32 products are exact in fp64 — everything else
// mul-then-add, no contraction), so results are bit-identical to it.
//
// What changes is where the chains run. A batch-32 step is a serial
// dependency chain of tiny phases, so one CTA leaves the SM's FP64 pipe and
// shared-memory port as the bound (~14 us per step). Here the units are split
// over the 4 CTAs of a cluster — CTA c owns layer-1 units J_c = [16c, 16c+16)
// and layer-2 units K_c = [8c, 8c+8) — and the activations the next phase
// needs in full move through distributed shared memory:
//   P0  x (all 32 records, every CTA)
//   F1  h1[:, J_c]  pushed to every CTA  -> cluster barrier
//   F2  h2[:, K_c]  pushed               -> cluster barrier
//   F3  logits / softmax / KL / d3 (all records, redundantly in every CTA)
//   B1  d2[:, K_c]  pushed               -> cluster barrier
//   B2  d1[:, J_c]
//   G   the gradient chains of the parameters CTA c owns (W0/b0 rows J_c,
//       W1/b1 rows K_c, W2 columns K_c, b2 on CTA 0, the loss everywhere)
//   SGD on the owned parameters; updated W1 / W2 / b2 entries pushed into the
//       other buffer of every CTA's (double-buffered) copies, ordered before
//       their use by the next step's first cluster barrier.
// Every CTA computes the identical loss, so all agree on divergence.
#include <cstddef>

#include "common.cuh"
#include "kernels.h"

namespace gbxcu {

#ifdef GBX_PHASE_TIMING
// Debug build only (tools/phase_timing.sh): per-phase cycle totals of CTA 0, thread 0.
__device__ unsigned long long g_cl_phase[16];
__device__ unsigned long long g_cl_t;
#define CL_MARK(i)                                                                             \
    do {                                                                                       \
        if (threadIdx.x == 0 && blockIdx.x == 0) {                                             \
            const unsigned long long t_ = clock64();                                           \
            if ((i) >= 0) g_cl_phase[(i) < 0 ? 0 : (i)] += t_ - g_cl_t;                        \
            g_cl_t = t_;                                                                       \
        }                                                                                      \
    } while (0)
#else
#define CL_MARK(i) ((void)0)
#endif

namespace {

constexpr int CL = TRAIN_CLUSTER;  // CTAs per cluster
constexpr int NTC = 512;           // threads per CTA
constexpr int TBR = 32;            // records per step
constexpr int J1 = H1 / CL;        // layer-1 units per CTA (16)
constexpr int K2 = H2 / CL;        // layer-2 units per CTA (8)
constexpr int W0S = F + 1;
constexpr int W1S = H1 + 1;
constexpr int WCS = J1 + 1;
constexpr int HS1 = H1 + 1;
constexpr int HS2 = H2 + 1;
constexpr int DS1 = J1 + 1;
// owned gradient chains: W0 rows (J1 x 44), b0 (J1), W1 rows (K2 x 64), b1 (K2),
// W2 columns (2 x K2), b2 (2, CTA 0), the loss
constexpr int Q_W0 = 0, Q_B0 = Q_W0 + J1 * F, Q_W1 = Q_B0 + J1, Q_B1 = Q_W1 + K2 * H1,
              Q_W2 = Q_B1 + K2, Q_B2 = Q_W2 + A * K2, Q_LOSS = Q_B2 + A, NQ = Q_LOSS + 1;
constexpr int QPT = (NQ + NTC - 1) / NTC;  // chains per thread (3)
static_assert(QPT == 3, "the G phase is written for three chains per thread");

struct ClSmem {
    double w0[J1 * W0S];   // own rows of W0: [jj][i]
    double b0[J1];
    double w1r[K2 * W1S];  // own rows of W1: [kk][j] (F2)
    double w1c[2][H2 * WCS];  // columns J_c of W1: [k][jj] (B2), double-buffered by step
    double b1[K2];
    double w2[2][A * H2];  // all of W2 (F3, B1), double-buffered by step
    double b2[2][A];
    // activations, double-buffered by step parity: every CTA pushes its own
    // columns into all four copies (distributed shared memory stores) before
    // the cluster barrier; a push of step s + 2 cannot reach a CTA still
    // reading step s's copy (three cluster barriers lie between them)
    double h1[2][TBR * HS1];  // all 64 columns
    double h2[2][TBR * HS2];  // all 32
    double d2[2][TBR * HS2];  // all 32
    double d1[TBR * DS1];  // own columns
    double d3[TBR * 2];
    double kl[TBR];
    double flag;           // 1: the step's loss sum is not finite
    double zero, one;      // operands of the G phase's dummy / bias chains
    uint32_t ord[2][TBR];  // record indices of the next two tiles (cp.async ring)
    alignas(16) double stage_t[2][TBR * 2];  // (16-byte cp.async destinations)
    alignas(16) float stage_f[2][TBR * F];
};
static_assert(offsetof(ClSmem, stage_t) % 16 == 0 && offsetof(ClSmem, stage_f) % 16 == 0, "cp.async alignment");

__device__ __forceinline__ void cl_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ uint32_t cl_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cl_addr(const void* local, uint32_t rank) {
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                 : "=r"(ra)
                 : "r"((uint32_t)__cvta_generic_to_shared(local)), "r"(rank));
    return ra;
}
// (volatile + memory clobber: never moved across the cluster barriers)
__device__ __forceinline__ void cl_st(double* local, uint32_t rank, double v) {
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(cl_addr(local, rank)), "d"(v) : "memory");
}

__device__ __forceinline__ void cp16(void* smem, const void* gmem, int src_bytes) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

__device__ __forceinline__ void cl_fetch_idx(ClSmem& S, int slot, const TrainArgs& a, size_t r0, int nv) {
    if ((int)threadIdx.x < nv) {
        const unsigned d = (unsigned)__cvta_generic_to_shared(&S.ord[slot][threadIdx.x]);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(a.order + r0 + threadIdx.x)
                     : "memory");
    }
}
__device__ __forceinline__ void cl_fetch_rows(ClSmem& S, int slot, const TrainArgs& a, int nv) {
    for (int t = threadIdx.x; t < TBR * (F / 4); t += NTC) {
        const int r = t / (F / 4), q = t - r * (F / 4);
        const float* src = a.feat;
        if (r < nv) src = a.feat + (size_t)S.ord[slot][r] * F + 4 * q;
        cp16(&S.stage_f[slot][r * F + 4 * q], src, r < nv ? 16 : 0);
    }
    if (threadIdx.x < TBR) {
        const int r = threadIdx.x;
        const double* src = a.tgt;
        if (r < nv) src = a.tgt + 2 * (size_t)S.ord[slot][r];
        cp16(&S.stage_t[slot][2 * r], src, r < nv ? 16 : 0);
    }
}

// the step's records [r0, r0 + nv): one tile per step (batch <= 32)
__device__ __forceinline__ bool cl_next(const TrainArgs& a, long n_steps, long& step, size_t& r0, int& nv) {
    if (r0 != (size_t)-1) ++step;
    if (step >= n_steps) return false;
    r0 = (size_t)step * (size_t)a.batch;
    nv = (int)min((size_t)a.batch, a.n - r0);
    return true;
}

// w = float(double(w) - lr * g) (policy.cpp:329-331), kept as fp64 in smem
__device__ __forceinline__ double cl_sgd(double w, double lr, double g) {
    return (double)__double2float_rn(__dsub_rn(w, __dmul_rn(lr, g)));
}

// flat parameter index of owned gradient chain q on CTA c (-1: not owned here)
__device__ __forceinline__ int cl_param_of(int q, int c) {
    if (q < Q_B0) return OFF_W0 + (c * J1 + q / F) * F + q % F;
    if (q < Q_W1) return OFF_B0 + c * J1 + (q - Q_B0);
    if (q < Q_B1) return OFF_W1 + (c * K2 + (q - Q_W1) / H1) * H1 + (q - Q_W1) % H1;
    if (q < Q_W2) return OFF_B1 + c * K2 + (q - Q_B1);
    if (q < Q_B2) return OFF_W2 + ((q - Q_W2) / K2) * H2 + c * K2 + (q - Q_W2) % K2;
    if (q < Q_LOSS) return c == 0 ? OFF_B2 + (q - Q_B2) : -1;
    return -1;  // the loss
}

}  // namespace

size_t train_cl_smem_bytes() { return sizeof(ClSmem); }

__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(NTC, 1) train_epoch_cluster_kernel(TrainArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ClSmem& S = *reinterpret_cast<ClSmem*>(smem_raw);
    const int tid = threadIdx.x;
    const int c = (int)cl_rank();
    if (*a.diverged_epoch >= 0) return;  // (uniform over the cluster)
    const long n_steps = (long)((a.n + a.batch - 1) / a.batch);

    // ---- prologue: index ring, the CTA's weight subsets, the first rows
    long s1 = 0, s2 = 0;
    size_t r1 = (size_t)-1, r2 = 0;
    int n1 = 0, n2 = 0;
    bool h1 = cl_next(a, n_steps, s1, r1, n1);
    if (h1) cl_fetch_idx(S, 0, a, r1, n1);
    s2 = s1;
    r2 = r1;
    bool h2 = h1 && cl_next(a, n_steps, s2, r2, n2);
    if (h2) cl_fetch_idx(S, 1, a, r2, n2);
    cp_commit();
    for (int t = tid; t < J1 * F; t += NTC) {
        const int jj = t / F, i = t - jj * F;
        S.w0[jj * W0S + i] = (double)a.params[OFF_W0 + (c * J1 + jj) * F + i];
    }
    if (tid < J1) S.b0[tid] = (double)a.params[OFF_B0 + c * J1 + tid];
    for (int t = tid; t < K2 * H1; t += NTC) {
        const int kk = t / H1, j = t - kk * H1;
        S.w1r[kk * W1S + j] = (double)a.params[OFF_W1 + (c * K2 + kk) * H1 + j];
    }
    for (int t = tid; t < H2 * J1; t += NTC) {
        const int k = t / J1, jj = t - k * J1;
        S.w1c[0][k * WCS + jj] = (double)a.params[OFF_W1 + k * H1 + c * J1 + jj];
    }
    if (tid < K2) S.b1[tid] = (double)a.params[OFF_B1 + c * K2 + tid];
    if (tid < A * H2) S.w2[0][tid] = (double)a.params[OFF_W2 + tid];
    if (tid < A) S.b2[0][tid] = (double)a.params[OFF_B2 + tid];
    if (tid == 0) {
        S.zero = 0.0;
        S.one = 1.0;
    }
    cp_wait();
    __syncthreads();
    if (h1) cl_fetch_rows(S, 0, a, n1);
    cp_commit();
    h1 = h2; s1 = s2; r1 = r2; n1 = n2;
    s2 = s1; r2 = r1;
    h2 = h1 && cl_next(a, n_steps, s2, r2, n2);

    double g[QPT];
#pragma unroll
    for (int m = 0; m < QPT; ++m) g[m] = 0.0;
    double epoch_total = 0.0;  // CTA 0, the thread holding the loss chain
    int wb = 0;                // buffer of the W1-column / W2 / b2 copies the next step reads
    cl_sync();                 // every CTA of the cluster is running before any DSMEM access
    CL_MARK(-1);

    for (long step = 0; step < n_steps; ++step) {
        const int k = (int)(step & 1);
        const size_t r0 = (size_t)step * (size_t)a.batch;
        const int nv = (int)min((size_t)a.batch, a.n - r0);
        const double nb = (double)nv;            // |b| (single rank: the step's records)
        const double inv_b = 1.0 / nb;           // batch_kl_gradient's 1/|b|
        cp_wait();                               // this thread's copies: step's rows, next indices
        __syncthreads();
        if (h1) cl_fetch_rows(S, k ^ 1, a, n1);  // rows of the next step
        if (h2) cl_fetch_idx(S, k, a, r2, n2);   // indices of the step after
        cp_commit();
        h1 = h2; s1 = s2; r1 = r2; n1 = n2;
        if (h2) h2 = cl_next(a, n_steps, s2, r2, n2);

        CL_MARK(0);  // step top (wait, prefetch issue)
        // ---- P0: the step's features and targets are read in place from the
        //      staging slot (features widened per use, exactly); the step-top
        //      barrier made them visible
        const float* xs = S.stage_f[k];
        const double* tg = S.stage_t[k];

        CL_MARK(1);  // P0
        // ---- F1: h1[r][16c + jj] = relu(b0 + sum_i w0[j][i] x[r][i]), DFMA chain over i
        {
            const int r = tid >> 4, jj = tid & 15;
            double acc = S.b0[jj];
            const double* wr = S.w0 + jj * W0S;
            const float* xr = xs + r * F;
#pragma unroll
            for (int i = 0; i < F; ++i) acc = fma(wr[i], (double)xr[i], acc);  // fp32 x fp32 exact in fp64
            const double h = acc > 0.0 ? acc : 0.0;
            double* dst = &S.h1[k][r * HS1 + c * J1 + jj];
            *dst = h;
#pragma unroll
            for (int o = 1; o < CL; ++o) cl_st(dst, (uint32_t)((c + o) % CL), h);
        }
        CL_MARK(2);  // F1
        cl_sync();
        CL_MARK(3);  // barrier 1
        CL_MARK(4);  // gather h1
        // ---- F2: h2[r][8c + kk] = relu(b1 + sum_j w1[k][j] h1[r][j]), mul-then-add
        if (tid < TBR * K2) {
            const int r = tid >> 3, kk = tid & 7;
            double acc = S.b1[kk];
            const double* wr = S.w1r + kk * W1S;
            const double* hr = S.h1[k] + r * HS1;
#pragma unroll 16
            for (int j = 0; j < H1; ++j) acc = madd_rn(acc, wr[j], hr[j]);
            const double h = acc > 0.0 ? acc : 0.0;
            double* dst = &S.h2[k][r * HS2 + c * K2 + kk];
            *dst = h;
#pragma unroll
            for (int o = 1; o < CL; ++o) cl_st(dst, (uint32_t)((c + o) % CL), h);
        }
        cl_sync();

        CL_MARK(5);  // F2 + barrier 2 + gather h2
        // ---- F3 (all records, identical in every CTA) + B1 (own columns)
        if (tid < 2 * TBR) {
            const int r = tid >> 1, a2 = tid & 1;
            double l = S.b2[wb][a2];
            const double* h = S.h2[k] + r * HS2;
            const double* wr = S.w2[wb] + a2 * H2;
#pragma unroll 8
            for (int kx = 0; kx < H2; ++kx) l = madd_rn(l, wr[kx], h[kx]);
            const double lo = __shfl_xor_sync(0xffffffffu, l, 1);
            const double l0 = a2 ? lo : l, l1 = a2 ? l : lo;
            const double m = l0 < l1 ? l1 : l0;  // std::max(l0, l1)
            const double e = exp(__dsub_rn(l, m));
            const double eo = __shfl_xor_sync(0xffffffffu, e, 1);
            const double s = a2 ? __dadd_rn(eo, e) : __dadd_rn(e, eo);  // e0 + e1
            const double p = __ddiv_rn(e, s);
            const double pc = clampp(p);
            const double tc = clampp(tg[2 * r + a2]);
            const double lr = log(__ddiv_rn(pc, tc));
            const double term = __dmul_rn(pc, lr);
            const double to = __shfl_xor_sync(0xffffffffu, term, 1);
            const double loss = __dadd_rn(__dadd_rn(0.0, a2 ? to : term), a2 ? term : to);
            const bool valid = r < nv;
            if (a2 == 0) S.kl[r] = valid ? loss : 0.0;
            const double d3 = valid ? __dmul_rn(__dmul_rn(p, __dsub_rn(lr, loss)), inv_b) : 0.0;
            S.d3[2 * r + a2] = d3;
            // B1: d2[r][k] = (0 + d3_0 w2_0k) + d3_1 w2_1k, masked by h2 > 0;
            //     thread a2 covers own columns kk in [4 a2, 4 a2 + 4)
            const double d3o = __shfl_xor_sync(0xffffffffu, d3, 1);
            const double d30 = a2 ? d3o : d3, d31 = a2 ? d3 : d3o;
#pragma unroll
            for (int q = 0; q < K2 / 2; ++q) {
                const int kx = c * K2 + (K2 / 2) * a2 + q;
                double d = madd_rn(0.0, d30, S.w2[wb][kx]);
                d = madd_rn(d, d31, S.w2[wb][H2 + kx]);
                const double dv = h[kx] <= 0.0 ? 0.0 : d;
                double* dst = &S.d2[k][r * HS2 + kx];
                *dst = dv;
#pragma unroll
                for (int o = 1; o < CL; ++o) cl_st(dst, (uint32_t)((c + o) % CL), dv);
            }
        }
        cl_sync();

        CL_MARK(6);  // F3 + B1 + barrier 3 + gather d2
        // ---- B2: d1[r][jj] = sum_k d2[r][k] w1[k][16c + jj], masked by h1 > 0
        {
            const int r = tid >> 4, jj = tid & 15;
            double acc = 0.0;
            const double* dr = S.d2[k] + r * HS2;
#pragma unroll
            for (int kx = 0; kx < H2; ++kx) acc = madd_rn(acc, dr[kx], S.w1c[wb][kx * WCS + jj]);
            S.d1[r * DS1 + jj] = S.h1[k][r * HS1 + c * J1 + jj] <= 0.0 ? 0.0 : acc;
        }
        __syncthreads();
        // (no cluster barrier: the SGD below writes the OTHER copy buffer, which
        //  every CTA last read a step ago — before this step's first barrier)

        CL_MARK(7);  // B2
        // ---- G: the owned parameters' gradient chains, records in batch order,
        //      the thread's (up to 3) chains interleaved. Every chain is
        //      acc = acc + (A[r] * B[r]) with B = 1.0 for the bias / loss sums
        //      (a * 1.0 == a exactly, so this IS acc + a). All 32 rows: a padding
        //      row's d1 / d2 / d3 / kl are +0, which leave every accumulator
        //      unchanged (they start at +0 and can never become -0).
        {
            const double* pa[QPT];
            const double* pb[QPT];
            const float* px[QPT];  // W0 chains: B = the fp32 features (widened exactly)
            int sa[QPT], sb[QPT];
#pragma unroll
            for (int m = 0; m < QPT; ++m) {
                const int q = tid + m * NTC;
                pa[m] = &S.zero;  // (not owned here: a dummy chain of zeros)
                pb[m] = &S.one;
                px[m] = nullptr;
                sa[m] = sb[m] = 0;
                if (q < Q_B0) {
                    const int jj = q / F, i = q - jj * F;
                    pa[m] = S.d1 + jj; sa[m] = DS1;
                    px[m] = xs + i; sb[m] = F;
                } else if (q < Q_W1) {
                    pa[m] = S.d1 + (q - Q_B0); sa[m] = DS1;
                } else if (q < Q_B1) {
                    const int kk = (q - Q_W1) / H1, j = (q - Q_W1) % H1;
                    pa[m] = S.d2[k] + c * K2 + kk; sa[m] = HS2;
                    pb[m] = S.h1[k] + j; sb[m] = HS1;
                } else if (q < Q_W2) {
                    pa[m] = S.d2[k] + c * K2 + (q - Q_B1); sa[m] = HS2;
                } else if (q < Q_B2) {
                    const int a2 = (q - Q_W2) / K2, kk = (q - Q_W2) % K2;
                    pa[m] = S.d3 + a2; sa[m] = 2;
                    pb[m] = S.h2[k] + c * K2 + kk; sb[m] = HS2;
                } else if (q < Q_LOSS) {
                    if (c == 0) { pa[m] = S.d3 + (q - Q_B2); sa[m] = 2; }
                } else if (q == Q_LOSS) {
                    pa[m] = S.kl; sa[m] = 1;
                }
            }
            // chain 0 is a W0 chain on every thread (Q_B0 > NTC), chain 1 on
            // threads < Q_B0 - NTC (whole warps), chain 2 never
            static_assert(Q_B0 >= NTC && Q_B0 - NTC <= NTC && (Q_B0 - NTC) % 32 == 0 && 2 * NTC >= Q_B0,
                          "W0 chain layout");
            if (tid < Q_B0 - NTC) {
#pragma unroll
                for (int r = 0; r < TBR; ++r) {
                    g[0] = madd_rn(g[0], pa[0][r * sa[0]], (double)px[0][r * F]);
                    g[1] = madd_rn(g[1], pa[1][r * sa[1]], (double)px[1][r * F]);
                    g[2] = madd_rn(g[2], pa[2][r * sa[2]], pb[2][r * sb[2]]);
                }
            } else {
#pragma unroll
                for (int r = 0; r < TBR; ++r) {
                    g[0] = madd_rn(g[0], pa[0][r * sa[0]], (double)px[0][r * F]);
                    g[1] = madd_rn(g[1], pa[1][r * sa[1]], pb[1][r * sb[1]]);
                    g[2] = madd_rn(g[2], pa[2][r * sa[2]], pb[2][r * sb[2]]);
                }
            }
#pragma unroll
            for (int m = 0; m < QPT; ++m)
                if (tid + m * NTC == Q_LOSS) S.flag = isfinite(g[m]) ? 0.0 : 1.0;  // loss finite iff the sum is
        }
        __syncthreads();
        if (S.flag != 0.0) {  // identical on every CTA: all leave at the same step
            if (c == 0 && tid == 0) *a.diverged_epoch = a.epoch;
            break;
        }
        CL_MARK(8);  // G + flag
        // ---- SGD on the owned parameters, new W1 / W2 / b2 entries into every copy
#pragma unroll
        for (int m = 0; m < QPT; ++m) {
            const int q = tid + m * NTC;
            if (q >= NQ) continue;
            if (q == Q_LOSS) {
                if (c == 0) epoch_total = madd_rn(epoch_total, __ddiv_rn(g[m], nb), nb);
            } else if (q < Q_B0) {
                const int jj = q / F, i = q - jj * F;
                S.w0[jj * W0S + i] = cl_sgd(S.w0[jj * W0S + i], a.lr, g[m]);
            } else if (q < Q_W1) {
                S.b0[q - Q_B0] = cl_sgd(S.b0[q - Q_B0], a.lr, g[m]);
            } else if (q < Q_B1) {
                const int kk = (q - Q_W1) / H1, j = (q - Q_W1) % H1;
                const double w = cl_sgd(S.w1r[kk * W1S + j], a.lr, g[m]);
                S.w1r[kk * W1S + j] = w;
                // next step's column copy of the CTA owning unit j (B2 there)
                const uint32_t oc = (uint32_t)(j / J1);
                double* dst = &S.w1c[wb ^ 1][(c * K2 + kk) * WCS + (j - (int)oc * J1)];
                if ((int)oc == c) *dst = w;
                else cl_st(dst, oc, w);
            } else if (q < Q_W2) {
                S.b1[q - Q_B1] = cl_sgd(S.b1[q - Q_B1], a.lr, g[m]);
            } else if (q < Q_B2) {
                const int a2 = (q - Q_W2) / K2, kk = (q - Q_W2) % K2;
                const int idx = a2 * H2 + c * K2 + kk;
                const double w = cl_sgd(S.w2[wb][idx], a.lr, g[m]);
                S.w2[wb ^ 1][idx] = w;
                for (int o = 1; o < CL; ++o) cl_st(&S.w2[wb ^ 1][idx], (uint32_t)((c + o) % CL), w);
            } else if (c == 0) {
                const int a2 = q - Q_B2;
                const double w = cl_sgd(S.b2[wb][a2], a.lr, g[m]);
                S.b2[wb ^ 1][a2] = w;
                for (int o = 1; o < CL; ++o) cl_st(&S.b2[wb ^ 1][a2], (uint32_t)o, w);
            }
            g[m] = 0.0;
        }
        wb ^= 1;
        CL_MARK(9);  // SGD + pushes
        // (the next step's first cluster barrier orders the pushes before
        //  F3 / B2 read them; this CTA's own updates before its next F1 / F2
        //  by the step-top barrier)
    }
    cp_wait();
    cl_sync();  // no CTA leaves while a peer may still write into its copies
    // epoch loss = total / n (policy.cpp:334); owned params back to global
    if (c == 0 && tid == Q_LOSS % NTC && *a.diverged_epoch < 0)
        a.epoch_loss[a.epoch] = __ddiv_rn(epoch_total, (double)a.n);
    for (int q = tid; q < NQ; q += NTC) {
        const int p = cl_param_of(q, c);
        if (p < 0) continue;
        double v;
        if (q < Q_B0) v = S.w0[(q / F) * W0S + q % F];
        else if (q < Q_W1) v = S.b0[q - Q_B0];
        else if (q < Q_B1) v = S.w1r[((q - Q_W1) / H1) * W1S + (q - Q_W1) % H1];
        else if (q < Q_W2) v = S.b1[q - Q_B1];
        else if (q < Q_B2) v = S.w2[wb][((q - Q_W2) / K2) * H2 + c * K2 + (q - Q_W2) % K2];
        else v = S.b2[wb][q - Q_B2];
        a.params[p] = (float)v;
    }
}

}  // namespace gbxcu

#ifdef GBX_PHASE_TIMING
extern "C" int gbxcu_debug_phase_cycles_cl(unsigned long long* out, int reset) {
    if (cudaMemcpyFromSymbol(out, gbxcu::g_cl_phase, sizeof(unsigned long long) * 16) != cudaSuccess) return 3;
    if (reset) {
        unsigned long long z[16] = {};
        cudaMemcpyToSymbol(gbxcu::g_cl_phase, z, sizeof(z));
    }
    return 0;
}
#endif
