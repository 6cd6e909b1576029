// k_wide.cu — the wide-MLP (C4: 44 -> H -> H -> 2, H = 512) training path on
// the 5th-generation tensor cores (tcgen05, kind::tf32, fp32 accumulation in
// TMEM).
//
// The reference hard-codes 44-64-32-2 (proj/include/gbx/policy.hpp:32-35);
// BASELINE.json config C4 asks for a hidden-512 variant on a bf16/TF32
// tensor-core path. Semantics follow fit / run_forward / accumulate_gradient
// generalised over widths (oracle/gbx_oracle.c restates them for any dims);
// parity is tolerance-based ("parity unpinned" by the reference).
//
// One training step = five TN GEMMs (both operands K-major) with fused
// epilogues plus a CUDA-core head:
//   G1  H1  = relu(X W0^T + b0)       [B x 512]  (X gathered through the epoch permutation)
//   G2  H2  = relu(H1 W1^T + b1)      [B x 512]
//   head logits = H2 W2^T + b2, softmax, KL, d3, D2 = (d3 W2) . [H2 > 0]
//   G3  D1  = (D2 W1) . [H1 > 0]      [B x 512]  (B operand = W1^T copy)
//   G4  gW1 = D2^T H1                 [512 x 512], K = batch, split-K
//   G5  gW0 = D1^T X                  [512 x 48],  K = batch, split-K
// Transposed activations needed as K-major operands of G4/G5 are written by
// the producing epilogues (a TMEM row is one batch record, so writing the
// transpose is a coalesced store across the warp).
#include <cuda.h>

#include <cstddef>

#include "common.cuh"
#include "kernels.h"
#include "tc_util.cuh"

namespace gbxcu {

using namespace tc;

constexpr int GM = 128;      // rows per CTA tile (TMEM lanes)
constexpr int GN = 128;      // columns per CTA tile (TMEM columns)
constexpr int GK = 32;       // K per pipeline stage (4 x kind::tf32 K=8)
constexpr int GSTAGES = 3;
constexpr int GTHREADS = 128;

struct GemmSmem {
    float a[GSTAGES][GK / 4][GM][4];  // canonical K-major: [chunk][row][4]
    float b[GSTAGES][GK / 4][GN][4];
    uint64_t mbar[GSTAGES];
    uint64_t done;
    uint32_t tmem;
};

size_t gemm_smem_bytes() { return sizeof(GemmSmem); }

// Stage loader: rows [row0, row0+GM) of A (optionally gathered through a_rows)
// and [col0, col0+GN) of B, K range [k0, k0+GK). Out-of-range rows/columns and
// K >= Kdim are zero-filled (cp.async src-size 0). lda/ldb in floats, multiples of 4.
__device__ __forceinline__ void gemm_load_stage(GemmSmem& S, int slot, const GemmArgs& g, int row0,
                                                int col0, int k0) {
    constexpr int CH = GK / 4;  // 16-byte chunks per row per stage
    for (int t = threadIdx.x; t < GM * CH; t += GTHREADS) {
        const int r = t / CH, c = t % CH;
        const int row = row0 + r, k = k0 + 4 * c;
        const bool ok = row < g.M && k < g.K;
        const float* src = g.A;
        if (ok) {
            const size_t ar = g.a_rows ? (size_t)g.a_rows[row] : (size_t)row;
            src = g.A + ar * (size_t)g.lda + k;
        }
        cp_async16(&S.a[slot][c][r][0], src, ok ? 16 : 0);
    }
    for (int t = threadIdx.x; t < GN * CH; t += GTHREADS) {
        const int r = t / CH, c = t % CH;
        const int col = col0 + r, k = k0 + 4 * c;
        const bool ok = col < g.N && k < g.K;
        const float* src = ok ? g.B + (size_t)col * g.ldb + k : g.B;
        cp_async16(&S.b[slot][c][r][0], src, ok ? 16 : 0);
    }
    cp_async_commit_group();
}

// Epilogue for 16 consecutive output columns [c0, c0+16) of one row (the
// calling thread's TMEM lane). Full, 16-byte aligned chunks use 128-bit
// loads/stores (each thread moves 64 contiguous bytes per chunk).
__device__ __forceinline__ bool chunk_vec_ok(const void* base, size_t ld, int c0, int n) {
    return c0 + 16 <= n && (ld % 4) == 0 && ((uintptr_t)base % 16) == 0;
}

__device__ __forceinline__ void gemm_epilogue(const GemmArgs& g, int row, bool row_ok, int c0,
                                              const float (&v)[16]) {
    if (!row_ok) return;
    switch (g.epi) {
        case EPI_STORE: {  // split-K partial (or plain) row-major store
            float* o = g.out + (size_t)blockIdx.z * g.split_stride + (size_t)row * g.ldo;
            if (chunk_vec_ok(g.out, g.ldo, c0, g.N) && (g.split_stride % 4) == 0) {
                float4* o4 = reinterpret_cast<float4*>(o + c0);
#pragma unroll
                for (int q = 0; q < 4; ++q) o4[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
            } else {
#pragma unroll
                for (int i = 0; i < 16; ++i)
                    if (c0 + i < g.N) o[c0 + i] = v[i];
            }
            break;
        }
        case EPI_BIAS_RELU: {  // h = relu(acc + bias): row-major and/or transposed
            if (chunk_vec_ok(g.bias, 0, c0, g.N) && (!g.out || chunk_vec_ok(g.out, g.ldo, c0, g.N))) {
                float h[16];
                const float4* b4 = reinterpret_cast<const float4*>(g.bias + c0);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float4 b = __ldg(b4 + q);
                    const float z0 = v[4 * q] + b.x, z1 = v[4 * q + 1] + b.y, z2 = v[4 * q + 2] + b.z,
                                z3 = v[4 * q + 3] + b.w;
                    h[4 * q] = z0 > 0.f ? z0 : 0.f;
                    h[4 * q + 1] = z1 > 0.f ? z1 : 0.f;
                    h[4 * q + 2] = z2 > 0.f ? z2 : 0.f;
                    h[4 * q + 3] = z3 > 0.f ? z3 : 0.f;
                }
                if (g.out) {
                    float4* o4 = reinterpret_cast<float4*>(g.out + (size_t)row * g.ldo + c0);
#pragma unroll
                    for (int q = 0; q < 4; ++q) o4[q] = make_float4(h[4 * q], h[4 * q + 1], h[4 * q + 2], h[4 * q + 3]);
                }
                if (g.out_t) {
#pragma unroll
                    for (int i = 0; i < 16; ++i) g.out_t[(size_t)(c0 + i) * g.ldt + row] = h[i];
                }
                break;
            }
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int c = c0 + i;
                if (c >= g.N) break;
                const float z = v[i] + g.bias[c];
                const float h = z > 0.f ? z : 0.f;
                if (g.out) g.out[(size_t)row * g.ldo + c] = h;
                if (g.out_t) g.out_t[(size_t)c * g.ldt + row] = h;
            }
            break;
        }
        case EPI_MASK_T: {  // d = acc * [mask > 0], transposed store
            if (chunk_vec_ok(g.mask, g.ldm, c0, g.N)) {
                const float4* m4 = reinterpret_cast<const float4*>(g.mask + (size_t)row * g.ldm + c0);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float4 m = __ldg(m4 + q);
                    const float mk[4] = {m.x, m.y, m.z, m.w};
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        g.out_t[(size_t)(c0 + 4 * q + j) * g.ldt + row] = mk[j] > 0.f ? v[4 * q + j] : 0.f;
                }
                break;
            }
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int c = c0 + i;
                if (c >= g.N) break;
                const float d = g.mask[(size_t)row * g.ldm + c] > 0.f ? v[i] : 0.f;
                g.out_t[(size_t)c * g.ldt + row] = d;
            }
            break;
        }
        default: break;
    }
}

// D[M x N] = A[M x K] . B[N x K]^T (+ epilogue). Grid: (ceil(N/GN), ceil(M/GM), splits).
__global__ void __launch_bounds__(GTHREADS) tc_gemm_kernel(GemmArgs g) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    GemmSmem& S = *reinterpret_cast<GemmSmem*>(smem_raw);
    const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
    const int col0 = blockIdx.x * GN, row0 = blockIdx.y * GM;
    // split-K: this CTA covers K blocks [kb_lo, kb_hi)
    const int nkb = (g.K + GK - 1) / GK;
    const int per = (nkb + gridDim.z - 1) / gridDim.z;
    const int kb_lo = blockIdx.z * per, kb_hi = min(nkb, kb_lo + per);

    if (w == 0) tmem_alloc(&S.tmem, GN);
    if (tid == 0) {
        for (int s = 0; s < GSTAGES; ++s) mbar_init(&S.mbar[s], 1);
        mbar_init(&S.done, 1);
        fence_mbar_init();
    }
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t tacc = S.tmem;
    const uint32_t idesc = idesc_tf32(GM, GN);

    // prologue: first GSTAGES-1 stages in flight
    for (int s = 0; s < GSTAGES - 1; ++s) {
        if (kb_lo + s < kb_hi) gemm_load_stage(S, s, g, row0, col0, (kb_lo + s) * GK);
        else cp_async_commit_group();
    }
    uint32_t phase_bits = 0;  // per-slot mbarrier parity
    for (int kb = kb_lo; kb < kb_hi; ++kb) {
        const int it = kb - kb_lo, slot = it % GSTAGES;
        // queue stage it+GSTAGES-1 into the slot the MMA of iteration it-1 read
        const int nxt = it + GSTAGES - 1, nslot = nxt % GSTAGES;
        if (kb_lo + nxt < kb_hi) {
            if (it >= 1) {
                mbar_wait(&S.mbar[nslot], (phase_bits >> nslot) & 1);
                phase_bits ^= 1u << nslot;
            }
            gemm_load_stage(S, nslot, g, row0, col0, (kb_lo + nxt) * GK);
        } else {
            cp_async_commit_group();
        }
        cp_async_wait_group<GSTAGES - 1>();
        fence_async_smem();
        __syncthreads();
        if (tid == 0) {
            fence_after_sync();
            const uint32_t a0 = smem_u32(&S.a[slot][0][0][0]), b0 = smem_u32(&S.b[slot][0][0][0]);
#pragma unroll
            for (int s = 0; s < GK / 8; ++s) {
                const uint64_t ad = smem_desc(a0 + 2 * s * GM * 16, GM * 16, 128);
                const uint64_t bd = smem_desc(b0 + 2 * s * GN * 16, GN * 16, 128);
                mma_tf32(tacc, ad, bd, idesc, (it > 0 || s > 0) ? 1u : 0u);
            }
            commit_to(&S.mbar[slot]);
        }
    }
    // drain: the last commit's barrier completes after every earlier MMA
    if (tid == 0) commit_to(&S.done);
    mbar_wait(&S.done, 0);
    fence_after_sync();
    cp_async_wait_group<0>();

    const int row = row0 + 32 * w + lane;
    for (int c0 = 0; c0 < GN; c0 += 16) {
        float v[16];
        tmem_ld16(tacc + ((uint32_t)(32 * w) << 16) + c0, v);
        tmem_ld_wait();
        if (kb_hi <= kb_lo) {
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = 0.f;
        }
        gemm_epilogue(g, row, row < g.M, col0 + c0, v);
    }
    fence_before_sync();
    __syncthreads();
    if (w == 0) tmem_dealloc(tacc, GN);
}

// ------------------------------------------------ TMA-pipelined GEMM (tcgen05)
// D[M x N] = A[M x K] . B[N x K]^T with both operands K-major in global
// memory, staged by TMA as {32 fp32 = 128 B, rows} boxes with the 128-byte
// swizzle (one box per operand per stage; UMMA descriptors SWIZZLE_128B,
// SBO = 8 rows x 128 B, K advanced 32 B per kind::tf32 K=8 step), a 4-stage
// mbarrier ring, and warp specialisation:
//   warp 0 lane 0 : TMA producer (waits "empty", arms "full" with the bytes)
//   warp 1 lane 0 : MMA issuer (waits "full", 4 x kind::tf32 K=8, commit -> "empty")
//   warps 0..3    : epilogue (TMEM -> registers -> fused epilogue -> global)
// Out-of-range rows / K are zero-filled by TMA. Tile BM=128 x BN, BK=32.
constexpr int TM_BM = 128, TM_BK = 32, TM_STAGES = 4;

template <int BN>
struct TmaSmem {
    // [stage][row][32 fp32] with the 128-byte swizzle (TMA writes it, UMMA reads it)
    float a[TM_STAGES][TM_BM * TM_BK];
    float b[TM_STAGES][BN * TM_BK];
    uint64_t full[TM_STAGES];
    uint64_t empty[TM_STAGES];
    uint64_t done;
    uint32_t tmem;
};

template <int BN>
size_t tma_gemm_smem_bytes() { return sizeof(TmaSmem<BN>) + 1024; }
template size_t tma_gemm_smem_bytes<64>();
template size_t tma_gemm_smem_bytes<128>();
template size_t tma_gemm_smem_bytes<256>();

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* mbar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(mbar)), "r"(bytes)
                 : "memory");
}
// bounded wait: a protocol bug must not hang the GPU (traps after ~seconds)
__device__ __forceinline__ void mbar_wait_bounded(uint64_t* mbar, uint32_t parity) {
    uint32_t done = 0;
    for (uint32_t it = 0; !done; ++it) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}\n"
            : "=r"(done)
            : "r"(smem_u32(mbar)), "r"(parity)
            : "memory");
        if (it > (1u << 28)) __trap();
    }
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* mbar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(mbar))
        : "memory");
}

template <int BN>
__global__ void __launch_bounds__(128, 1)
tma_gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                GemmArgs g) {
    extern __shared__ unsigned char smem_raw[];
    // 1024-B alignment for the operand tiles
    TmaSmem<BN>& S = *reinterpret_cast<TmaSmem<BN>*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
    const int col0 = blockIdx.x * BN, row0 = blockIdx.y * TM_BM;
    const int nkb = (g.K + TM_BK - 1) / TM_BK;
    const int per = (nkb + gridDim.z - 1) / gridDim.z;
    const int kb_lo = blockIdx.z * per, kb_hi = min(nkb, kb_lo + per);
    const int nk = max(0, kb_hi - kb_lo);

    if (w == 0) tmem_alloc(&S.tmem, BN);
    if (tid == 32) {
        for (int s = 0; s < TM_STAGES; ++s) {
            mbar_init(&S.full[s], 1);
            mbar_init(&S.empty[s], 1);
        }
        mbar_init(&S.done, 1);
        fence_mbar_init();
    }
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t tacc = S.tmem;

    if (tid == 0) {
        // ---- TMA producer
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_b) : "memory");
        constexpr uint32_t bytes = (TM_BM + BN) * TM_BK * 4;
        for (int it = 0; it < nk; ++it) {
            const int slot = it % TM_STAGES;
            if (it >= TM_STAGES) mbar_wait_bounded(&S.empty[slot], ((it / TM_STAGES) - 1) & 1);
            mbar_arrive_expect_tx(&S.full[slot], bytes);
            const int k0 = (kb_lo + it) * TM_BK;
            tma_load_2d(&S.a[slot][0], &map_a, k0, row0, &S.full[slot]);
            tma_load_2d(&S.b[slot][0], &map_b, k0, col0, &S.full[slot]);
        }
    } else if (tid == 32) {
        // ---- MMA issuer
        const uint32_t idesc = idesc_tf32(TM_BM, BN);
        for (int it = 0; it < nk; ++it) {
            const int slot = it % TM_STAGES;
            mbar_wait_bounded(&S.full[slot], (it / TM_STAGES) & 1);
            fence_after_sync();
            const uint32_t a0 = smem_u32(&S.a[slot][0]), b0 = smem_u32(&S.b[slot][0]);
#pragma unroll
            for (int s = 0; s < TM_BK / 8; ++s) {
                const uint64_t ad = smem_desc_sw128(a0 + 32 * s);
                const uint64_t bd = smem_desc_sw128(b0 + 32 * s);
                mma_tf32(tacc, ad, bd, idesc, (it > 0 || s > 0) ? 1u : 0u);
            }
            commit_to(&S.empty[slot]);  // frees the stage once these MMAs have read it
        }
        commit_to(&S.done);  // after every MMA issued above
    }
    __syncwarp();
    // ---- epilogue (all 4 warps): one TMEM lane (= output row) per thread
    if (nk > 0) mbar_wait_bounded(&S.done, 0);
    fence_after_sync();
    const int row = row0 + 32 * w + lane;
    for (int c0 = 0; c0 < BN; c0 += 16) {
        float v[16];
        tmem_ld16(tacc + ((uint32_t)(32 * w) << 16) + c0, v);
        tmem_ld_wait();
        if (nk == 0) {
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = 0.f;
        }
        gemm_epilogue(g, row, row < g.M, col0 + c0, v);
    }
    fence_before_sync();
    __syncthreads();
    if (w == 0) tmem_dealloc(tacc, BN);
}

template __global__ void tma_gemm_kernel<64>(const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap, GemmArgs);
template __global__ void tma_gemm_kernel<128>(const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap, GemmArgs);
template __global__ void tma_gemm_kernel<256>(const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap, GemmArgs);

// ----------------------------------------------------------- CUDA-core parts
// XT[i][r] = feat[rows[r]][i] for i < 44, zeros for 44 <= i < 48 (K-major B
// operand of the gW0 GEMM).
__global__ void wide_gather_xt_kernel(const float* __restrict__ feat, const uint32_t* __restrict__ rows,
                                      int nb, float* __restrict__ xt, int ldt, float* __restrict__ xg) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nb) return;
    const float4* x = reinterpret_cast<const float4*>(feat + (size_t)rows[r] * F);
    float4 v[F / 4];
#pragma unroll
    for (int q = 0; q < F / 4; ++q) v[q] = __ldg(x + q);  // all 11 loads in flight
    // gathered rows, K padded to 48 (TMA operand of the first GEMM)
    float4* g4 = reinterpret_cast<float4*>(xg + (size_t)r * 48);
#pragma unroll
    for (int q = 0; q < F / 4; ++q) g4[q] = v[q];
    g4[F / 4] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int q = 0; q < F / 4; ++q) {
        xt[(size_t)(4 * q) * ldt + r] = v[q].x;
        xt[(size_t)(4 * q + 1) * ldt + r] = v[q].y;
        xt[(size_t)(4 * q + 2) * ldt + r] = v[q].z;
        xt[(size_t)(4 * q + 3) * ldt + r] = v[q].w;
    }
    xt[(size_t)F * ldt + r] = 1.f;  // ones row: column 44 of D1^T X is gb0
#pragma unroll
    for (int i = F + 1; i < 48; ++i) xt[(size_t)i * ldt + r] = 0.f;
}

// Head: one warp per record, 32 records per block (1024 threads). logits =
// b2 + H2 w2^T (fp64 sums), softmax, KL with the reference clamps, d3 = p
// (ln(p^/t^) - L) / |b|, D2 = (d3 w2) [H2>0] written row-major, and
// transposed through a shared-memory tile (coalesced 128-byte column runs);
// per-record KL and d3 kept for the reductions. Requires hidden <= 1024.
__global__ void __launch_bounds__(1024) wide_head_kernel(WideHeadArgs a) {
    extern __shared__ float tile[];  // [32 records][hidden + 1]
    __shared__ float sd3[32][2];
    __shared__ double skl[32];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const int r0 = blockIdx.x * 32, r = r0 + wl, Hd = a.hidden, ts = Hd + 1;
    if (r < a.nb) {
        const float* h = a.h2 + (size_t)r * Hd;
        double l0 = 0.0, l1 = 0.0;
        for (int k = lane; k < Hd; k += 32) {
            const double hv = h[k];
            l0 += (double)a.w2[k] * hv;
            l1 += (double)a.w2[Hd + k] * hv;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            l0 += __shfl_xor_sync(0xffffffffu, l0, o);
            l1 += __shfl_xor_sync(0xffffffffu, l1, o);
        }
        l0 += a.b2[0];
        l1 += a.b2[1];
        const double m = l0 < l1 ? l1 : l0;
        const double e0 = exp(l0 - m), e1 = exp(l1 - m);
        const double p0 = e0 / (e0 + e1), p1 = e1 / (e0 + e1);
        const size_t rec = a.rows ? a.rows[r] : (size_t)r;
        const double pc0 = clampp(p0), pc1 = clampp(p1);
        const double lr0 = log(pc0 / clampp(a.tgt[2 * rec])), lr1 = log(pc1 / clampp(a.tgt[2 * rec + 1]));
        const double loss = pc0 * lr0 + pc1 * lr1;
        const double d30 = p0 * (lr0 - loss) * a.inv_b, d31 = p1 * (lr1 - loss) * a.inv_b;
        if (lane == 0) {
            a.kl[r] = loss;
            a.d3[2 * r] = (float)d30;
            a.d3[2 * r + 1] = (float)d31;
            sd3[wl][0] = (float)d30;
            sd3[wl][1] = (float)d31;
            skl[wl] = loss;
        }
        for (int k = lane; k < Hd; k += 32) {
            const float d = h[k] > 0.f ? (float)(d30 * (double)a.w2[k] + d31 * (double)a.w2[Hd + k]) : 0.f;
            a.d2[(size_t)r * Hd + k] = d;
            tile[wl * ts + k] = d;
        }
    } else if (lane == 0) {
        sd3[wl][0] = sd3[wl][1] = 0.f;
        skl[wl] = 0.0;
    }
    __syncthreads();
    // block partials (fixed record order): gW2[a][k] = sum d3[r][a] H2[r][k],
    // gb1[k] = sum D2[r][k]; gb2, KL sums by thread 0
    const int nr = min(32, a.nb - r0);
    double* prow = a.part + (size_t)blockIdx.x * (3 * Hd + 3);
    for (int k = threadIdx.x; k < Hd; k += blockDim.x) {
        double g0 = 0.0, g1 = 0.0, gb = 0.0;
        for (int q = 0; q < nr; ++q) {
            const double hv = a.h2[(size_t)(r0 + q) * Hd + k];
            g0 += (double)sd3[q][0] * hv;
            g1 += (double)sd3[q][1] * hv;
            gb += tile[q * ts + k];
        }
        prow[k] = g0;
        prow[Hd + k] = g1;
        prow[2 * Hd + k] = gb;
    }
    if (threadIdx.x == 0) {
        double s0 = 0.0, s1 = 0.0, sl = 0.0;
        for (int q = 0; q < nr; ++q) {
            s0 += sd3[q][0];
            s1 += sd3[q][1];
            sl += skl[q];
        }
        prow[3 * Hd] = s0;
        prow[3 * Hd + 1] = s1;
        prow[3 * Hd + 2] = sl;
    }
    // transposed store: warp wl writes columns k = wl, wl + 32, ...; lane = record
    if (r0 + lane < a.nb)
        for (int k = wl; k < Hd; k += 32) a.d2t[(size_t)k * a.ldt + r0 + lane] = tile[lane * ts + k];
}

// out[j] = sum_r in[j][r] (fixed-shape tree per row; one block per row).
__global__ void row_sum_kernel(const float* __restrict__ in, int ld, int ncols, float* __restrict__ out) {
    __shared__ double red[32];
    const float* row = in + (size_t)blockIdx.x * ld;
    double s4[4] = {0.0, 0.0, 0.0, 0.0};
    int c = threadIdx.x;
    for (; c + 3 * (int)blockDim.x < ncols; c += 4 * blockDim.x) {
        float v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = __ldg(row + c + j * blockDim.x);  // 4 loads in flight
#pragma unroll
        for (int j = 0; j < 4; ++j) s4[j] += v[j];
    }
    for (; c < ncols; c += blockDim.x) s4[0] += row[c];
    double s = (s4[0] + s4[1]) + (s4[2] + s4[3]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) out[blockIdx.x] = (float)s;
    }
}

// gW2[a][k] = sum_r d3[r][a] H2[r][k], gb2[a] = sum_r d3[r][a], loss = sum_r kl[r]:
// grid (ceil(H/64), RSPLIT), block (64 columns, 4 record lanes); each thread
// keeps 4 loads in flight; fixed-order partials reduced by split_reduce_f64.
__global__ void __launch_bounds__(256) wide_w2_partial_kernel(const float* __restrict__ h2,
                                                              const float* __restrict__ d3,
                                                              const double* __restrict__ kl, int nb,
                                                              int hidden, double* __restrict__ part) {
    __shared__ double red[4][64][2];
    __shared__ double sc[4][3];
    const int cx = threadIdx.x & 63, ry = threadIdx.x >> 6;
    const int k = blockIdx.x * 64 + cx;
    const int per = (nb + gridDim.y - 1) / gridDim.y;
    const int r0 = blockIdx.y * per, r1 = min(nb, r0 + per);
    double s0 = 0, s1 = 0, g0 = 0, g1 = 0, ls = 0;
    int r = r0 + ry;
    for (; r + 12 < r1; r += 16) {
        float hv[4];
        float2 dv[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            hv[j] = k < hidden ? __ldg(h2 + (size_t)(r + 4 * j) * hidden + k) : 0.f;
            dv[j] = __ldg(reinterpret_cast<const float2*>(d3) + r + 4 * j);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            s0 += (double)dv[j].x * hv[j];
            s1 += (double)dv[j].y * hv[j];
            if (cx == 0) {
                g0 += dv[j].x;
                g1 += dv[j].y;
                ls += kl[r + 4 * j];
            }
        }
    }
    for (; r < r1; r += 4) {
        const float2 dv = __ldg(reinterpret_cast<const float2*>(d3) + r);
        const float hv = k < hidden ? __ldg(h2 + (size_t)r * hidden + k) : 0.f;
        s0 += (double)dv.x * hv;
        s1 += (double)dv.y * hv;
        if (cx == 0) {
            g0 += dv.x;
            g1 += dv.y;
            ls += kl[r];
        }
    }
    red[ry][cx][0] = s0;
    red[ry][cx][1] = s1;
    if (cx == 0) {
        sc[ry][0] = g0;
        sc[ry][1] = g1;
        sc[ry][2] = ls;
    }
    __syncthreads();
    double* o = part + (size_t)blockIdx.y * (2 * hidden + 3);
    if (ry == 0 && k < hidden) {
        o[k] = (red[0][cx][0] + red[1][cx][0]) + (red[2][cx][0] + red[3][cx][0]);
        o[hidden + k] = (red[0][cx][1] + red[1][cx][1]) + (red[2][cx][1] + red[3][cx][1]);
    }
    if (blockIdx.x == 0 && threadIdx.x < 3) {
        const int q = threadIdx.x;
        o[2 * hidden + q] = (sc[0][q] + sc[1][q]) + (sc[2][q] + sc[3][q]);
    }
}

// Sum split partials in order: dst[i] = sum_s src[s * stride + i] (fp32 or fp64 src).
__global__ void split_reduce_f32_kernel(const float* __restrict__ src, int splits, size_t stride,
                                        int rows, int cols, int ld_src, float* __restrict__ dst,
                                        int ld_dst) {
    const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (size_t)rows * cols) return;
    const int r = (int)(t / cols), c = (int)(t % cols);
    float s = 0.f;
    for (int q = 0; q < splits; ++q) s += src[q * stride + (size_t)r * ld_src + c];
    dst[(size_t)r * ld_dst + c] = s;
}

__global__ void split_reduce_f64_kernel(const double* __restrict__ src, int splits, int n,
                                        float* __restrict__ dst, double* __restrict__ loss_out) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    double s = 0.0;
    int q = 0;
    for (; q + 3 < splits; q += 4) {
        double v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = src[(size_t)(q + j) * n + t];
#pragma unroll
        for (int j = 0; j < 4; ++j) s += v[j];
    }
    for (; q < splits; ++q) s += src[(size_t)q * n + t];
    if (t == n - 1) *loss_out = s;  // last slot is the KL sum
    else dst[t] = (float)s;
}

// SGD over the flat generic-layout params, W1^T refresh, divergence check.
// grad/params in serialization order: w0[H][44] b0[H] w1[H][H] b1[H] w2[2][H] b2[2].
__global__ void wide_update_kernel(float* __restrict__ params, const float* __restrict__ grad,
                                   const double* __restrict__ loss_sum, size_t nb, double lr,
                                   int hidden, float* __restrict__ w1t, float* __restrict__ w0p,
                                   const int* __restrict__ epoch, int* __restrict__ diverged,
                                   double* __restrict__ epoch_acc, size_t np) {
    if (*diverged >= 0) return;
    const double loss = *loss_sum / (double)nb;
    if (!isfinite(loss)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) *diverged = *epoch;
        return;
    }
    const size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p == 0) *epoch_acc += loss * (double)nb;
    if (p >= np) return;
    const float nw = __double2float_rn((double)params[p] - lr * (double)grad[p]);
    params[p] = nw;
    const size_t w1_off = (size_t)hidden * F + hidden;
    if (p >= w1_off && p < w1_off + (size_t)hidden * hidden) {
        const size_t t = p - w1_off, k = t / hidden, j = t % hidden;
        w1t[j * hidden + k] = nw;
    } else if (p < (size_t)hidden * F) {
        w0p[(p / F) * 48 + p % F] = nw;  // K-padded W0 (first GEMM's B operand)
    }
}

// W1^T and the K-padded W0 [H][48] from the flat params (initial copies).
__global__ void wide_w1t_kernel(const float* __restrict__ params, int hidden, float* __restrict__ w1t,
                                float* __restrict__ w0p) {
    const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < (size_t)hidden * 48) {
        const size_t j = t / 48, i = t % 48;
        w0p[t] = i < F ? params[j * F + i] : 0.f;
    }
    if (t >= (size_t)hidden * hidden) return;
    const size_t w1_off = (size_t)hidden * F + hidden, k = t / hidden, j = t % hidden;
    w1t[j * hidden + k] = params[w1_off + t];
}

// PolicyNet::init generalised to dims {44, H, H, 2} (proj/src/policy.cpp:128-139).
__global__ void wide_init_kernel(uint64_t seed, int hidden, float* __restrict__ params, size_t np) {
    const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= np) return;
    const size_t H = hidden;
    const size_t o_b0 = H * F, o_w1 = o_b0 + H, o_b1 = o_w1 + H * H, o_w2 = o_b1 + H, o_b2 = o_w2 + 2 * H;
    int l;
    size_t k;
    if (t < o_b0) { l = 0; k = t; }
    else if (t < o_w1) { params[t] = 0.f; return; }
    else if (t < o_b1) { l = 1; k = t - o_w1; }
    else if (t < o_w2) { params[t] = 0.f; return; }
    else if (t < o_b2) { l = 2; k = t - o_w2; }
    else { params[t] = 0.f; return; }
    const int fan[4] = {F, hidden, hidden, A};
    const double bound = sqrt(6.0 / (double)(fan[l] + fan[l + 1]));
    const uint64_t s = derive_seed3(seed, 0x1A17u, (uint64_t)l);
    params[t] = __double2float_rn(__dmul_rn(signed_unit_of(sm_draw(s, (uint64_t)k + 1)), bound));
}

// Forward head for inference: probabilities from H2 (fp64 sums), one warp per row.
__global__ void wide_probs_kernel(const float* __restrict__ h2, const float* __restrict__ w2,
                                  const float* __restrict__ b2, int nb, int hidden,
                                  double* __restrict__ probs) {
    const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (r >= nb) return;
    double l0 = 0.0, l1 = 0.0;
    for (int k = lane; k < hidden; k += 32) {
        const double hv = h2[(size_t)r * hidden + k];
        l0 += (double)w2[k] * hv;
        l1 += (double)w2[hidden + k] * hv;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        l0 += __shfl_xor_sync(0xffffffffu, l0, o);
        l1 += __shfl_xor_sync(0xffffffffu, l1, o);
    }
    if (lane == 0) {
        l0 += b2[0];
        l1 += b2[1];
        const double m = l0 < l1 ? l1 : l0;
        const double e0 = exp(l0 - m), e1 = exp(l1 - m);
        probs[2 * (size_t)r] = e0 / (e0 + e1);
        probs[2 * (size_t)r + 1] = e1 / (e0 + e1);
    }
}

// Zero columns [c_lo, c_hi) of a [rows][ld] matrix (K tail of the transposed
// activations, so 16-byte K chunks that straddle the batch end read zeros).
__global__ void zero_cols_kernel(float* __restrict__ m, int rows, int ld, int c_lo, int c_hi) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int w = c_hi - c_lo;
    if (w <= 0 || t >= rows * w) return;
    m[(size_t)(t / w) * ld + c_lo + t % w] = 0.f;
}

// gW0 [H][48] split partials -> flat grad w0 block [H][44]; column 44 (the
// ones row of X^T) -> gb0.
__global__ void wide_gw0_kernel(const float* __restrict__ src, int splits, size_t stride, int hidden,
                                float* __restrict__ dst, float* __restrict__ gb0) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= hidden * (F + 1)) return;
    const int j = t / (F + 1), i = t % (F + 1);
    float s = 0.f;
    for (int q = 0; q < splits; ++q) s += src[q * stride + (size_t)j * 48 + i];
    if (i < F) dst[j * F + i] = s;
    else gb0[j] = s;
}

// Sum the head's block partials in block order: grid ceil(W/32), block (32
// columns x 8 block groups), 4 loads in flight per thread.
__global__ void __launch_bounds__(256) wide_head_reduce_kernel(const double* __restrict__ part, int nblocks,
                                                               int hidden, float* __restrict__ gw2,
                                                               float* __restrict__ gb2, float* __restrict__ gb1,
                                                               double* __restrict__ loss_out) {
    __shared__ double red[8][32];
    const int W = 3 * hidden + 3;
    const int cx = threadIdx.x & 31, gy = threadIdx.x >> 5;
    const int col = blockIdx.x * 32 + cx;
    double s = 0.0;
    if (col < W) {
        int b = gy;
        for (; b + 24 < nblocks; b += 32) {
            double v[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) v[j] = part[(size_t)(b + 8 * j) * W + col];
#pragma unroll
            for (int j = 0; j < 4; ++j) s += v[j];
        }
        for (; b < nblocks; b += 8) s += part[(size_t)b * W + col];
    }
    red[gy][cx] = s;
    __syncthreads();
    if (gy == 0 && col < W) {
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) t += red[q][cx];
        if (col < 2 * hidden) gw2[col] = (float)t;
        else if (col < 3 * hidden) gb1[col - 2 * hidden] = (float)t;
        else if (col < 3 * hidden + 2) gb2[col - 3 * hidden] = (float)t;
        else *loss_out = t;
    }
}

}  // namespace gbxcu
