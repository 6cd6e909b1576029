// k_wide16.cu — the wide-MLP (C4: 44 -> H -> H -> 2, H = 512) training step on
// the 5th-generation tensor cores with BF16 operands (tcgen05 kind::f16, fp32
// accumulation in TMEM): twice the TF32 path's tensor rate and half its
// operand bytes.
//
// Semantics: fit / run_forward / accumulate_gradient generalised over widths
// (the reference hard-codes 44-64-32-2, proj/include/gbx/policy.hpp:32-35;
// oracle/gbx_oracle.c restates them for any dims). Activations are stored in
// BF16 between the GEMMs; the master parameters, biases, the head (logits,
// softmax, KL, d3) and the update w = float(double(w) - lr g) stay fp32/fp64.
// oracle/wide_emul.py models these rounding points for the parity tests.
//
// One step = 5 GEMMs (both operands K-major, staged by TMA with the 128-byte
// swizzle into an mbarrier ring; one producer thread, one MMA-issuing thread,
// four epilogue warps reading TMEM) + a gather and a fused update:
//   gather  Xg = bf16(X[rows]) [B][64], X^T [64][B] (row 44 = 1: gb0 via G5)
//   G1  H1 = relu(Xg W0^T + b0)            -> H1 [B][H], H1^T [H][B]     (BN 256)
//   G2  acc = H1 W1^T, full rows (BN = H): the head runs in the epilogue:
//       h2 = relu(acc + b1) (never stored), logits (fp64), softmax, KL, d3,
//       D2 = (d3 w2) [h2 > 0] -> D2 [B][H], D2^T [H][B];
//       per-CTA column sums gW2 = sum d3 h2, gb1 = sum D2, gb2, KL
//   G3  D1 = (D2 W1) [H1 > 0]              -> D1^T [H][B]               (BN 256)
//   G4  gW1 = D2^T H1 (K = batch, split-K fp32 partials)
//   G5  gW0 | gb0 = D1^T [X | 1] (K = batch, split-K fp32 partials)
//   update: every gradient reduced in a fixed order, loss / divergence, SGD,
//       refreshed BF16 copies of W0, W1, W1^T — one launch.
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstddef>

#include "common.cuh"
#include "kernels.h"
#include "tc_util.cuh"

namespace gbxcu {

using namespace tc;

#ifdef GBX_PHASE_TIMING
// Debug build only (tools/phase_timing.sh): per-launch timeline of the first
// eight steps of a fit — slot = step * 8 + launch (0 gather, 1..5 G1..G5,
// 6 update); points 0 entry, 1 inputs ready (after griddepcontrol.wait),
// 2 main loop done, 3 exit; {min, max} over the CTAs (globaltimer ns).
__device__ unsigned long long g_w16_tr[64][8][2];  // points 4..7: epilogue phases (head / SGD)
__device__ unsigned long long g_w16_steps[4096];  // every step: first gather CTA entry
#define W16_TR(slot, pt)                                                          \
    do {                                                                          \
        if ((slot) >= 0 && threadIdx.x == 0) {                                    \
            unsigned long long t_;                                                \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                \
            atomicMin(&g_w16_tr[slot][pt][0], t_);                                \
            atomicMax(&g_w16_tr[slot][pt][1], t_);                                \
        }                                                                         \
    } while (0)
#else
#define W16_TR(slot, pt) \
    do {                 \
    } while (0)
#endif

namespace {

constexpr int W_BM = 128;  // rows per CTA tile (TMEM lanes)
constexpr int W_BK = 64;   // bf16 per 128-byte swizzle row = K per stage

// Instruction descriptor: A, B = BF16 (K-major), D = F32, dense.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
    return (1u << 4)                       // c_format = F32
           | (1u << 7)                     // a_format = BF16
           | (1u << 10)                    // b_format = BF16
           | ((uint32_t)(N >> 3) << 17)    // n_dim
           | ((uint32_t)(M >> 4) << 24);   // m_dim
}

// MN-major operand with the 128-byte swizzle: TMA boxes of {64 elements along
// M/N (128 B), 64 K rows}, so a K row of 64 M/N elements is one 128-byte row,
// 8 K rows form a 1024-byte swizzle atom (SBO), and the next 64 M/N elements
// are the next box, 8 KB on (LBO). K steps of 16 advance the start 2 KB.
__device__ __forceinline__ uint64_t smem_desc_mn128(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)(8192 >> 4) << 16;    // LBO: next 64-element M/N chunk
    d |= (uint64_t)(1024 >> 4) << 32;    // SBO: next 8 K rows
    d |= (uint64_t)1 << 46;              // version = 1 (Blackwell)
    d |= (uint64_t)2 << 61;              // SWIZZLE_128B
    return d;
}
constexpr uint32_t IDESC_A_MN = 1u << 15, IDESC_B_MN = 1u << 16;

__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void mbar_expect(uint64_t* mbar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(mbar)), "r"(bytes)
                 : "memory");
}
// bounded wait: a protocol bug must not hang the GPU (traps after ~seconds)
__device__ __forceinline__ void mbar_wait_b(uint64_t* mbar, uint32_t parity) {
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
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* mbar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(mbar))
        : "memory");
}

// TMA tensor store shared -> global (bulk-group completion), issued by one thread.
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(map), "r"(c0),
                 "r"(c1), "r"(smem_u32(src))
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// at most one committed group still reading its shared-memory source
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
// every committed group complete (writes performed)
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// generic-proxy shared-memory writes -> visible to the TMA (async proxy)
__device__ __forceinline__ void fence_proxy_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Warp-collective: 32 consecutive fp32 columns of this warp's 32 TMEM lanes.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
          "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// Programmatic dependent launch: let the next kernel of the step start its
// prologue (TMEM / barrier setup) now; wait for the previous kernel's results.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Thread-block cluster (the fused head's CTA pair): barrier and a read of
// the peer CTA's shared memory (distributed shared memory).
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// split form: loads issued between the two are not held up by the release
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ double ld_peer_f64(const double* local, uint32_t peer) {
    uint32_t a = smem_u32(local), ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(peer));
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(ra) : "memory");
    return v;
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    const __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&v);
}
__device__ __forceinline__ void load_row16(const __nv_bfloat16* src, float (&m)[16]) {
    const uint4 q0 = __ldg(reinterpret_cast<const uint4*>(src));
    const uint4 q1 = __ldg(reinterpret_cast<const uint4*>(src) + 1);
    const uint32_t w[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const __nv_bfloat162 v = *reinterpret_cast<const __nv_bfloat162*>(&w[i]);
        m[2 * i] = __bfloat162float(v.x);
        m[2 * i + 1] = __bfloat162float(v.y);
    }
}

template <int BN, int ST>
struct W16Smem {
    __nv_bfloat16 a[ST][W_BM * W_BK];  // [stage][row][64] with the 128-byte swizzle
    __nv_bfloat16 b[ST][BN * W_BK];
    uint64_t full[ST];
    uint64_t empty[ST];
    uint64_t done;
    uint32_t tmem;
};

__host__ __device__ constexpr int tmem_cols(int bn) { return bn <= 32 ? 32 : bn <= 64 ? 64 : bn <= 128 ? 128 : bn <= 256 ? 256 : 512; }

// Epilogue warps per TMEM lane quarter (w_ew<EPI>(), kernels.h): warp w reads
// lanes 32 (w % 4).., column group w / 4. (32 warps for the head measured
// slower: 64 registers per thread spill, and the larger shared-memory
// footprint slowed the launches that follow the GEMMs.)
constexpr int W_EW_MAX = 4;

// Epilogue output staging (per warp, double-buffered over its 16-column
// chunks): the chunk's 32 rows x 16 columns in bf16, row-major ([32][16], one
// 32-byte row per lane) and transposed ([16][32], a 64-byte row per column),
// written to global memory by two TMA tensor stores (full 32-byte sectors,
// no per-lane address streams).
struct OutStage {
    __nv_bfloat16 rm[2][32 * 16];
    __nv_bfloat16 tr[2][16 * 32];
};
constexpr size_t OUT_STAGE_BYTES = 4 * W_EW_MAX * sizeof(OutStage);
struct HeadScratch {
    float b1[W16_MAX_H];
    float w2[2][W16_MAX_H];
    double w2d[2][W16_MAX_H];    // w2 widened once (the logits accumulate in fp64)
    double lg[W_EW_MAX][128][2];  // per column group: partial logits of the CTA's 128 rows
    double own[128][2];          // the CTA's partial logits (its columns), read by the pair peer
    double wsum[4][3][W16_MAX_H];  // per lane quarter: column sums (gW2_0, gW2_1, gb1)
    double red[4 * W_EW_MAX][3];
};


// Column sums of a warp's 32 rows: v[16] = this lane's (row's) values of 16
// columns; returns, in lanes l and l ^ 16, the sum over the 32 lanes of
// column l & 15 (recursive halving over lane bits 3..0, then bit 4: a fixed
// tree, 16 shuffles instead of a shared-memory round trip per row).
__device__ __forceinline__ float col_reduce16(float (&v)[16], int lane) {
#pragma unroll
    for (int b = 3, n = 8; b >= 0; --b, n >>= 1) {
        const bool hi = (lane >> b) & 1;
#pragma unroll
        for (int j = 0; j < n; ++j) {
            const float send = hi ? v[j] : v[j + n], keep = hi ? v[j + n] : v[j];
            v[j] = keep + __shfl_xor_sync(0xffffffffu, send, 1 << b);
        }
    }
    return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 16);
}

// One 16-column chunk of a warp's output (lane = row): stage it in bf16 and
// issue its TMA stores (row-major at (col, row0), transposed at (row0, col);
// RM / TR select which). Buffer k & 1 is reused two chunks later, after its
// previous stores have read it. Rows past M are clipped by the tensor maps.
__device__ __forceinline__ void stage_chunk(OutStage& o, int k, const float (&h)[16], const CUtensorMap* map_o,
                                            const CUtensorMap* map_ot, int col, int row0, int lane, bool RM,
                                            bool TR) {
    const int b = k & 1;
    if (k >= 2) {
        if (lane == 0) bulk_wait_read1();
        __syncwarp();
    }
    if (RM) {
        uint4* q = reinterpret_cast<uint4*>(o.rm[b] + lane * 16);
        q[0] = make_uint4(pack_bf16(h[0], h[1]), pack_bf16(h[2], h[3]), pack_bf16(h[4], h[5]), pack_bf16(h[6], h[7]));
        q[1] = make_uint4(pack_bf16(h[8], h[9]), pack_bf16(h[10], h[11]), pack_bf16(h[12], h[13]),
                          pack_bf16(h[14], h[15]));
    }
    if (TR) {
#pragma unroll
        for (int i = 0; i < 16; ++i) o.tr[b][i * 32 + lane] = __float2bfloat16_rn(h[i]);
    }
    fence_proxy_smem();
    __syncwarp();
    if (lane == 0) {
        if (RM) tma_store_2d(map_o, o.rm[b], col, row0);
        if (TR) tma_store_2d(map_ot, o.tr[b], row0, col);
        bulk_commit();
    }
}

}  // namespace

// the head keeps its scratch; its output staging follows it
__host__ __device__ constexpr size_t head_stage_off() { return (sizeof(HeadScratch) + 1023) & ~(size_t)1023; }

template <int BN, int ST>
size_t w16_gemm_smem_bytes() {
    size_t s = sizeof(W16Smem<BN, ST>);
    if (OUT_STAGE_BYTES > s) s = OUT_STAGE_BYTES;
    if (head_stage_off() + OUT_STAGE_BYTES > s) s = head_stage_off() + OUT_STAGE_BYTES;
    return s + 1024;
}
template size_t w16_gemm_smem_bytes<64, 6>();
template size_t w16_gemm_smem_bytes<128, 6>();
template size_t w16_gemm_smem_bytes<256, 4>();

// sum_q src[q * stride] in q order, sixteen loads in flight at a time
template <typename T>
__device__ __forceinline__ double ordered_sum(const T* __restrict__ src, size_t stride, int n) {
    double s = 0.0;
    for (int q = 0; q < n; q += 16) {
        T v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = q + j < n ? __ldg(src + (size_t)(q + j) * stride) : T(0);
#pragma unroll
        for (int j = 0; j < 16; ++j)
            if (q + j < n) s += v[j];
    }
    return s;
}

// Gradient of parameter p (serialization order w0[H][44] b0[H] w1[H][H]
// b1[H] w2[2][H] b2[2]) from the step's partials, summed in a fixed order.
__device__ __forceinline__ double w16_grad(const W16UpdArgs& u, size_t p) {
    const size_t H = u.hidden;
    const size_t o_b0 = H * F, o_w1 = o_b0 + H, o_b1 = o_w1 + H * H, o_w2 = o_b1 + H, o_b2 = o_w2 + 2 * H;
    const size_t hw = 3 * H + 3;
    if (p < o_w1) {  // gW0 | gb0: G5 partials [s5][H][64], column 44 = gb0
        const size_t j = p < o_b0 ? p / F : p - o_b0, i = p < o_b0 ? p % F : (size_t)F;
        return ordered_sum(u.p5 + j * 64 + i, H * 64, u.s5);
    }
    if (p < o_b1) return ordered_sum(u.p4 + (p - o_w1), H * H, u.s4);   // gW1: G4 partials [s4][H][H]
    if (p < o_w2) return ordered_sum(u.hp + 2 * H + (p - o_b1), hw, u.nhead);  // gb1
    if (p < o_b2) return ordered_sum(u.hp + (p - o_w2), hw, u.nhead);          // gW2
    return ordered_sum(u.hp + 3 * H + (p - o_b2), hw, u.nhead);                // gb2
}

// KL sum of the step over the head partials (warp 0; fixed lane order + tree:
// every block computes the identical value)
__device__ __forceinline__ double w16_kl_sum(const W16UpdArgs& u) {
    const int lane = threadIdx.x & 31;
    const size_t hw = 3 * (size_t)u.hidden + 3;
    double s = 0.0;
    for (int q = lane; q < u.nhead; q += 32) s += u.hp[(size_t)q * hw + 3 * u.hidden + 2];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}

// The fused softmax/KL head of G2 (see the kernel below), one CTA of a pair:
// TMEM accumulators at `tq` (this warp's lane quarter), the CTA's output
// columns [col0, col0 + BN). Also the tail of the fused G1+G2 launch.
template <int BN, int EW>
__device__ __forceinline__ void w16_head_epilogue(unsigned char* base, const W16Args& g, const CUtensorMap& map_o,
                                                  const CUtensorMap& map_ot, uint32_t tq, int col0, int row0,
                                                  double tg0, double tg1, float hb1, float hw20, float hw21) {
    constexpr int NTH = 128 * EW, CW = BN / EW;
    const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
    const int qw = w & 3, cg = w >> 2;
    const int rw0 = row0 + 32 * qw, row = rw0 + lane;
    const bool row_ok = row < g.M;
    const int cbeg = cg * CW;
    const uint32_t col0u = (uint32_t)col0;
    (void)col0u;
    // ---- fused head (G2). A CTA pair (thread-block cluster along x)
    //      covers full rows: each CTA its BN columns; the partial logits
    //      of its 4 column groups and of the pair combine in a fixed
    //      order (column group, then CTA) through (distributed) shared memory
    HeadScratch& T = *reinterpret_cast<HeadScratch*>(base);
    OutStage& O = reinterpret_cast<OutStage*>(base + head_stage_off())[w];
    const int H = g.N;
    static_assert(BN <= NTH, "one head column per thread");
    if (tid < BN && col0 + tid < H) {
        const int c = col0 + tid;
        T.b1[c] = hb1;
        T.w2[0][c] = hw20;
        T.w2[1][c] = hw21;
        T.w2d[0][c] = (double)hw20;
        T.w2d[1][c] = (double)hw21;
    }
    __syncthreads();
    const int cb = col0 + cbeg, cend = min(H, cb + CW);
    // pass 1: h2 = relu(acc + b1); partial logits in fp64 (two chains per output)
    double l0a = 0.0, l0b = 0.0, l1a = 0.0, l1b = 0.0;
    for (int c0 = cb; c0 < cend; c0 += 32) {
        float v[32];
        tmem_ld32(tq + (c0 - col0), v);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
            const float4 bb = *reinterpret_cast<const float4*>(&T.b1[c0 + i]);
            const double2 w0a = *reinterpret_cast<const double2*>(&T.w2d[0][c0 + i]);
            const double2 w0b = *reinterpret_cast<const double2*>(&T.w2d[0][c0 + i + 2]);
            const double2 w1a = *reinterpret_cast<const double2*>(&T.w2d[1][c0 + i]);
            const double2 w1b = *reinterpret_cast<const double2*>(&T.w2d[1][c0 + i + 2]);
            const float h0 = fmaxf(v[i] + bb.x, 0.f), h1 = fmaxf(v[i + 1] + bb.y, 0.f);
            const float h2 = fmaxf(v[i + 2] + bb.z, 0.f), h3 = fmaxf(v[i + 3] + bb.w, 0.f);
            l0a = fma((double)h0, w0a.x, l0a);
            l1a = fma((double)h0, w1a.x, l1a);
            l0b = fma((double)h1, w0a.y, l0b);
            l1b = fma((double)h1, w1a.y, l1b);
            l0a = fma((double)h2, w0b.x, l0a);
            l1a = fma((double)h2, w1b.x, l1a);
            l0b = fma((double)h3, w0b.y, l0b);
            l1b = fma((double)h3, w1b.y, l1b);
        }
    }
    T.lg[cg][32 * qw + lane][0] = l0a + l0b;
    T.lg[cg][32 * qw + lane][1] = l1a + l1b;
    W16_TR(g.dbg, 4);
    __syncthreads();
    const int rl = 32 * qw + lane;
    if (cg == 0) {
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int q = 0; q < EW; ++q) {
            s0 += T.lg[q][rl][0];
            s1 += T.lg[q][rl][1];
        }
        T.own[rl][0] = s0;
        T.own[rl][1] = s1;
    }
    const uint32_t crank = cluster_rank(), npair = (uint32_t)gridDim.x;  // 1 or 2 CTAs per row tile
    if (npair > 1) cluster_sync();  // the peer's partial logits are written
    else __syncthreads();
    // softmax, KL with the reference clamps, d3 = p (ln(p^/t^) - L) / |b|
    // (every column group of a row computes the same values)
    double d30 = 0.0, d31 = 0.0, loss = 0.0;
    {
        double s0 = T.own[rl][0], s1 = T.own[rl][1];
        if (npair > 1) {  // CTA 0's columns first
            const double p0 = ld_peer_f64(&T.own[rl][0], crank ^ 1u), p1 = ld_peer_f64(&T.own[rl][1], crank ^ 1u);
            if (crank == 0) {
                s0 += p0;
                s1 += p1;
            } else {
                s0 = p0 + s0;
                s1 = p1 + s1;
            }
        }
        if (row_ok) {
        const double z0 = (double)g.b2[0] + s0, z1 = (double)g.b2[1] + s1;
        const double m = z0 < z1 ? z1 : z0;
        const double e0 = exp(z0 - m), e1 = exp(z1 - m);
        const double p0 = e0 / (e0 + e1), p1 = e1 / (e0 + e1);
        const double pc0 = clampp(p0), pc1 = clampp(p1);
        const double lr0 = log(pc0 / clampp(tg0)), lr1 = log(pc1 / clampp(tg1));
        loss = pc0 * lr0 + pc1 * lr1;
        d30 = p0 * (lr0 - loss) * g.inv_b;
        d31 = p1 * (lr1 - loss) * g.inv_b;
        }
    }
    const float d3f0 = (float)d30, d3f1 = (float)d31;
    W16_TR(g.dbg, 5);
    // pass 2 (fp32): D2 = (d3 w2) [h2 > 0] -> D2 (row-major), D2^T (TMA
    // stores); column sums gW2 = sum d3 h2, gb1 = sum D2 over the warp's 32
    // rows (fp32 shuffle trees), per lane quarter in shared memory
    float vn[16];  // the next chunk's accumulators, loaded one chunk ahead
    tmem_ld16(tq + (cb - col0), vn);
    for (int c0 = cb; c0 < cend; c0 += 16) {
        float v[16], h[16], d[16];
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = vn[i];
        if (c0 + 16 < cend) tmem_ld16(tq + (c0 + 16 - col0), vn);
#pragma unroll
        for (int i = 0; i < 16; i += 4) {
            const float4 bb = *reinterpret_cast<const float4*>(&T.b1[c0 + i]);
            const float4 wa = *reinterpret_cast<const float4*>(&T.w2[0][c0 + i]);
            const float4 wb = *reinterpret_cast<const float4*>(&T.w2[1][c0 + i]);
            const float b4[4] = {bb.x, bb.y, bb.z, bb.w}, a4[4] = {wa.x, wa.y, wa.z, wa.w},
                        c4[4] = {wb.x, wb.y, wb.z, wb.w};
            // (packed fp32 pairs: each half rounds exactly like the scalar op)
#pragma unroll
            for (int j = 0; j < 4; j += 2) {
                const float2 s2v = __fadd2_rn(make_float2(v[i + j], v[i + j + 1]), make_float2(b4[j], b4[j + 1]));
                const float2 da = __fmul2_rn(make_float2(d3f0, d3f0), make_float2(a4[j], a4[j + 1]));
                const float2 dc = __fmul2_rn(make_float2(d3f1, d3f1), make_float2(c4[j], c4[j + 1]));
                const float2 dd = __fadd2_rn(da, dc);
                h[i + j] = row_ok ? fmaxf(s2v.x, 0.f) : 0.f;
                h[i + j + 1] = row_ok ? fmaxf(s2v.y, 0.f) : 0.f;
                d[i + j] = h[i + j] > 0.f ? dd.x : 0.f;
                d[i + j + 1] = h[i + j + 1] > 0.f ? dd.y : 0.f;
            }
        }
        stage_chunk(O, (c0 - cb) >> 4, d, &map_o, &map_ot, c0, rw0, lane, true, g.out_t != nullptr);
        float p[16];
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
            const float2 q = __fmul2_rn(make_float2(d3f0, d3f0), make_float2(h[i], h[i + 1]));
            p[i] = q.x;
            p[i + 1] = q.y;
        }
        const float s0 = col_reduce16(p, lane);
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
            const float2 q = __fmul2_rn(make_float2(d3f1, d3f1), make_float2(h[i], h[i + 1]));
            p[i] = q.x;
            p[i + 1] = q.y;
        }
        const float s1 = col_reduce16(p, lane);
        const float s2 = col_reduce16(d, lane);
        if (lane < 16) {
            T.wsum[qw][0][c0 + lane] = (double)s0;
            T.wsum[qw][1][c0 + lane] = (double)s1;
            T.wsum[qw][2][c0 + lane] = (double)s2;
        }
    }
    W16_TR(g.dbg, 6);
    // gb2 and KL of the rows (column group 0 only; fixed shuffle tree)
    const bool first = cg == 0 && crank == 0;
    double r0 = first ? d30 : 0.0, r1 = first ? d31 : 0.0, r2 = first ? loss : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        r0 += __shfl_xor_sync(0xffffffffu, r0, o);
        r1 += __shfl_xor_sync(0xffffffffu, r1, o);
        r2 += __shfl_xor_sync(0xffffffffu, r2, o);
    }
    if (lane == 0) {
        T.red[w][0] = r0;
        T.red[w][1] = r1;
        T.red[w][2] = r2;
    }
    __syncthreads();
    double* prow = g.head_part + (size_t)blockIdx.y * (3 * H + 3);
    for (int q = 0; q < 3; ++q)
        for (int c = col0 + tid; c < min(H, col0 + BN); c += NTH)
            prow[q * H + c] = ((T.wsum[0][q][c] + T.wsum[1][q][c]) + T.wsum[2][q][c]) + T.wsum[3][q][c];
    if (tid < 3 && crank == 0)
        prow[3 * H + tid] = ((T.red[0][tid] + T.red[1][tid]) + T.red[2][tid]) + T.red[3][tid];
    if (lane == 0) bulk_wait_all();
    if (npair > 1) cluster_sync();  // the peer has read this CTA's partial logits
}

// D[M x N] = A[M x K] . B[N x K]^T, bf16 operands, fp32 accumulation, epilogue EPI.
// Grid (ceil(N/BN), ceil(M/128), splits). Warp 0 lane 0: TMA producer; warp 1
// lane 0: MMA issuer; all 16 warps: epilogue (warp w: TMEM lanes 32 (w % 4)..
// = output rows, column group w / 4 of BN / 4 columns; thread = one row).
template <int BN, int ST, int EPI>
__global__ void __launch_bounds__(128 * w_ew<EPI>(), 1)
w16_gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                const __grid_constant__ CUtensorMap map_o, const __grid_constant__ CUtensorMap map_ot, W16Args g) {
    extern __shared__ unsigned char smem_raw[];
    unsigned char* base = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    W16Smem<BN, ST>& S = *reinterpret_cast<W16Smem<BN, ST>*>(base);
    constexpr int NMMA = BN > 256 ? 2 : 1;   // MMA N <= 256
    constexpr int MN = BN / NMMA;
    constexpr int BOX = BN > 256 ? 256 : BN;  // TMA box rows <= 256
    constexpr int TC = tmem_cols(BN);
    constexpr int EW = w_ew<EPI>(), NTH = 128 * EW;
    const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
    int col0 = blockIdx.x * BN, row0 = blockIdx.y * W_BM;
    // the fused SGD launch: tiles y < T1 are gW1 tiles (A = map_a, B = map_b),
    // the rest [gW0 | gb0] tiles (A = map_o, B = map_ot, 64 columns)
    const CUtensorMap* pma = &map_a;
    const CUtensorMap* pmb = &map_b;
    bool w0tile = false;
    if constexpr (EPI == W16_EPI_SGD) {
        const int nN = (g.N + BN - 1) / BN, T1 = ((g.M + W_BM - 1) / W_BM) * nN, t = blockIdx.y;
        if (t < T1) {
            row0 = (t / nN) * W_BM;
            col0 = (t % nN) * BN;
        } else {
            w0tile = true;
            row0 = (t - T1) * W_BM;
            col0 = 0;
            pma = &map_o;
            pmb = &map_ot;
        }
    }
    const int nkb = (g.K + W_BK - 1) / W_BK;
    const int per = (nkb + gridDim.z - 1) / gridDim.z;
    const int kb_lo = blockIdx.z * per, kb_hi = min(nkb, kb_lo + per);
    const int nk = max(0, kb_hi - kb_lo);

    W16_TR(g.dbg, 0);
    if (w == 0) tmem_alloc(&S.tmem, TC);
    if (tid == 32) {
        for (int s = 0; s < ST; ++s) {
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
    // (prologue done: the step's next kernel may start its own; every read of
    //  the previous kernel's results comes after its completion). G1 lets its
    //  successor launch only after its wait: the gather before it writes its
    //  Xg / X^T copy without waiting, so the chain of early launches must not
    //  run ahead to the gather two steps on (same copy) while this step's
    //  G4+G5 may still read it
    if constexpr (EPI == W16_EPI_H1) {
        pdl_wait();
        pdl_trigger();
    } else {
        pdl_trigger();
        pdl_wait();
    }
    W16_TR(g.dbg, 1);

    if (tid == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(pma) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(pmb) : "memory");
        if constexpr (EPI <= W16_EPI_D1T) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(&map_o) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(&map_ot) : "memory");
        }
        constexpr uint32_t bytes = (W_BM + BN) * W_BK * 2;
        for (int it = 0; it < nk; ++it) {
            const int slot = it % ST;
            if (it >= ST) mbar_wait_b(&S.empty[slot], ((it / ST) - 1) & 1);
            mbar_expect(&S.full[slot], bytes);
            const int k0 = (kb_lo + it) * W_BK;
            if constexpr (EPI == W16_EPI_SGD) {
                // MN-major operands (row-major D2 / H1 / D1 / Xg: K = records
                // are their rows): boxes of {64 M/N, 64 K}
#pragma unroll
                for (int h = 0; h < W_BM / 64; ++h) tma_2d(&S.a[slot][h * 64 * W_BK], pma, row0 + 64 * h, k0, &S.full[slot]);
#pragma unroll
                for (int h = 0; h < BN / 64; ++h) tma_2d(&S.b[slot][h * 64 * W_BK], pmb, col0 + 64 * h, k0, &S.full[slot]);
            } else if constexpr (EPI == W16_EPI_D1T) {
                // A = D2 K-major; B = W1 itself, MN-major ([j][k]: K = j its
                // rows), so no transposed copy of W1 is kept
                tma_2d(&S.a[slot][0], pma, k0, row0, &S.full[slot]);
#pragma unroll
                for (int h = 0; h < BN / 64; ++h) tma_2d(&S.b[slot][h * 64 * W_BK], pmb, col0 + 64 * h, k0, &S.full[slot]);
            } else {
                tma_2d(&S.a[slot][0], pma, k0, row0, &S.full[slot]);
#pragma unroll
                for (int h = 0; h < BN / BOX; ++h)
                    tma_2d(&S.b[slot][h * BOX * W_BK], pmb, k0, col0 + h * BOX, &S.full[slot]);
            }
        }
    } else if (tid == 32) {
        constexpr bool MNM = EPI == W16_EPI_SGD;  // MN-major A and B
        constexpr bool BMN = EPI == W16_EPI_D1T;  // K-major A, MN-major B
        const uint32_t idesc =
            idesc_bf16(W_BM, MN) | (MNM ? IDESC_A_MN | IDESC_B_MN : 0u) | (BMN ? IDESC_B_MN : 0u);
        for (int it = 0; it < nk; ++it) {
            const int slot = it % ST;
            mbar_wait_b(&S.full[slot], (it / ST) & 1);
            fence_after_sync();
            const uint32_t a0 = smem_u32(&S.a[slot][0]), b0 = smem_u32(&S.b[slot][0]);
#pragma unroll
            for (int s = 0; s < W_BK / 16; ++s) {  // K = 16 per MMA
                if constexpr (MNM) {  // 16 K rows of 128 B further
                    static_assert(NMMA == 1, "MN-major path: one MMA per K step");
                    mma_bf16(tacc, smem_desc_mn128(a0 + 2048 * s), smem_desc_mn128(b0 + 2048 * s), idesc,
                             (it > 0 || s > 0) ? 1u : 0u);
                } else if constexpr (BMN) {
                    static_assert(NMMA == 1, "MN-major B: one MMA per K step");
                    mma_bf16(tacc, smem_desc_sw128(a0 + 32 * s), smem_desc_mn128(b0 + 2048 * s), idesc,
                             (it > 0 || s > 0) ? 1u : 0u);
                } else {  // 32 B along the swizzled K-major row
                    const uint64_t ad = smem_desc_sw128(a0 + 32 * s);
#pragma unroll
                    for (int h = 0; h < NMMA; ++h) {
                        const uint64_t bd = smem_desc_sw128(b0 + h * MN * 128 + 32 * s);
                        mma_bf16(tacc + h * MN, ad, bd, idesc, (it > 0 || s > 0) ? 1u : 0u);
                    }
                }
            }
            commit_to(&S.empty[slot]);  // frees the stage once these MMAs have read it
        }
        commit_to(&S.done);
    }
    // (the head's targets: a gather through the record indices, issued while
    //  the MMAs run)
    double tg0 = 0.0, tg1 = 0.0;
    float hb1 = 0.f, hw20 = 0.f, hw21 = 0.f;  // (the head's b1 / w2 of column col0 + tid)
    if constexpr (EPI == W16_EPI_HEAD) {
        const int rr = row0 + 32 * (w & 3) + (tid & 31);
        if (rr < g.M) {
            const size_t rec = g.rows ? g.rows[rr] : (size_t)rr;
            tg0 = g.tgt[2 * rec];
            tg1 = g.tgt[2 * rec + 1];
        }
        if (tid < BN && col0 + tid < g.N) {
            hb1 = g.bias[col0 + tid];
            hw20 = g.w2[col0 + tid];
            hw21 = g.w2[g.N + col0 + tid];
        }
    }
    // (G3's mask — the stored bf16 H1 of this thread's row and 64 columns,
    //  written by G1, complete before this kernel's wait — loaded while the
    //  MMAs run)
    // (the fused SGD launch: the step's KL partials and the divergence flag,
    //  read by warp 2 while the MMAs run)
    double klv[2] = {0.0, 0.0};
    int dv = -1;
    if constexpr (EPI == W16_EPI_SGD) {
        if (w == 2) {
            const size_t hwd = 3 * (size_t)g.u.hidden + 3;
#pragma unroll
            for (int t = 0; t < 2; ++t)
                if (lane + 32 * t < g.u.nhead)
                    klv[t] = g.u.hp[(size_t)(lane + 32 * t) * hwd + 3 * g.u.hidden + 2];
            dv = *g.u.diverged;
        }
    }
    uint4 mk[EPI == W16_EPI_D1T ? 8 : 1];
    if constexpr (EPI == W16_EPI_D1T) {
        constexpr int CWm = BN / w_ew<EPI>();
        static_assert(CWm == 64, "mask prefetch: 64 columns per thread");
        const int rr = row0 + 32 * (w & 3) + (tid & 31), cb0 = col0 + (w >> 2) * CWm;
#pragma unroll
        for (int q = 0; q < 8; ++q) mk[q] = make_uint4(0u, 0u, 0u, 0u);
        if (rr < g.M && cb0 < g.N) {
            const uint4* src = reinterpret_cast<const uint4*>(g.mask + (size_t)rr * g.ldm + cb0);
#pragma unroll
            for (int q = 0; q < 8; ++q) mk[q] = __ldg(src + q);
        }
    }
    __syncwarp();
    if (nk > 0) mbar_wait_b(&S.done, 0);
    fence_after_sync();
    W16_TR(g.dbg, 2);

    const int qw = w & 3, cg = w >> 2;        // lane quarter, column group
    const int rw0 = row0 + 32 * qw;             // first row of this warp
    const int row = rw0 + lane;
    const bool row_ok = row < g.M;
    const uint32_t tq = tacc + ((uint32_t)(32 * qw) << 16);
    constexpr int CW = BN / EW;                 // columns per group
    const int cbeg = cg * CW;
    __syncthreads();  // every warp is past the mainloop: stage buffers are free for scratch

    if constexpr (EPI == W16_EPI_HEAD) {
        w16_head_epilogue<BN, EW>(base, g, map_o, map_ot, tq, col0, row0, tg0, tg1, hb1, hw20, hw21);
    } else if constexpr (EPI == W16_EPI_SGD) {
        // ---- fused split-K reduction + SGD (single-rank path). The S CTAs of
        //      a cluster (along z) hold the S K-split partials of one output
        //      tile; CTA cr sums its 128 / S rows of all S partials in split
        //      order (fp32 partials, fp64 sum: the update kernel's order) through
        //      distributed shared memory and applies SGD to them
        //      (policy.cpp:328-332), refreshing the bf16 operand copies (W1
        //      only: G3 reads it MN-major, no transposed copy). The
        //      gW1 and [gW0 | gb0] tiles share the launch; every thread of the
        //      grid also helps sum the head parameters' gradients (b1, W2, b2).
        W16_TR(g.dbg, 6);  // (probe: epilogue entry)
        const W16UpdArgs& u = g.u;
        constexpr int RS = BN + 4;  // padded fp32 row stride: conflict-free 16-byte stores
        constexpr int S = W16_SPLITS, B4 = BN / 4;
        constexpr int MAXG = (128 / S + 1) * B4 / NTH + 1;  // float4 groups per thread (upper bound)
        float* R = reinterpret_cast<float*>(base);
        double* sc = reinterpret_cast<double*>(R + 128 * RS);
        static_assert(128 * RS * 4 + 32 <= (int)sizeof(W16Smem<BN, ST>), "SGD scratch fits the ring");
        const int H = u.hidden;
        const size_t o_b0 = (size_t)H * F, o_w1 = o_b0 + H, o_b1 = o_w1 + (size_t)H * H;
        const int ncol = w0tile ? F + 1 : g.N;  // valid output columns
        // every global load of the epilogue is issued first (the step's KL
        // partials, the slice's old weights, the head partials) and consumed
        // after the TMEM dump: one round trip, overlapped with it
        const size_t hwd = 3 * (size_t)H + 3;
        // this CTA's rows of the tile: [r_lo, r_hi) (128 rows over S CTAs)
        const int cr = (int)cluster_rank();
        const int r_lo = cr * 128 / S, r_hi = (cr + 1) * 128 / S;
        const int n4 = (r_hi - r_lo) * B4;  // float4 groups of the slice
        for (int c0 = cbeg; c0 < cbeg + CW; c0 += 16) {
            float v[16];
            tmem_ld16(tq + c0, v);
            tmem_ld_wait();
            if (nk == 0) {
#pragma unroll
                for (int i = 0; i < 16; ++i) v[i] = 0.f;
            }
            float4* d = reinterpret_cast<float4*>(R + (32 * qw + lane) * RS + c0);
#pragma unroll
            for (int q = 0; q < 4; ++q) d[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        }
        W16_TR(g.dbg, 7);  // (probe: TMEM dumped)
        if (w == 2) {  // the step's loss: the KL partials in lane order + a fixed tree (w16_kl_sum)
            double kl = klv[0] + klv[1];
            for (int q = lane + 64; q < u.nhead; q += 32) kl += u.hp[(size_t)q * hwd + 3 * H + 2];  // (nhead > 64)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) kl += __shfl_xor_sync(0xffffffffu, kl, o);
            if (lane == 0) {
                sc[0] = kl / (double)u.nb;
                sc[1] = (double)dv;
            }
        }
        W16_TR(g.dbg, 4);
        // all S partials are in shared memory after this barrier; the
        // epilogue's global loads (old weights, head partials — used after the
        // exchange) go out between its arrive (whose release would otherwise
        // wait for them) and its wait
        cluster_arrive();
        float wold[MAXG][4];
#pragma unroll
        for (int t = 0; t < MAXG; ++t) {
            const int idx = tid + t * NTH, j = row0 + r_lo + idx / B4;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int kl = 4 * (idx % B4) + e;
                wold[t][e] = 0.f;
                if (idx >= n4 || j >= g.M || col0 + kl >= ncol) continue;
                wold[t][e] = w0tile ? u.params[kl < F ? (size_t)j * F + kl : o_b0 + j]
                                    : u.params[o_w1 + (size_t)j * H + col0 + kl];
            }
        }
        // head parameter gradients: four threads per parameter, each summing a
        // quarter of the row tiles' head partials, combined in a fixed tree
        const size_t nh = u.np - o_b1;
        // (spread over every CTA — the first 64 threads of each — so no cluster
        //  waits on a CTA carrying many of these loads)
        const size_t ncta = (size_t)gridDim.x * gridDim.y * gridDim.z;
        const size_t HT = ((4 * nh + ncta - 1) / ncta + 3) & ~(size_t)3;  // head threads per CTA (<= 4 * 386 / 12)
        const size_t cta = ((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
        const size_t gt = (size_t)tid < HT ? cta * HT + tid : ~(size_t)0 >> 2;
        const size_t ph = o_b1 + gt / 4;
        constexpr int HQ = 16;  // head partial rows per thread (nhead <= 64 in one batch)
        double hv[HQ];
        int q0 = 0, q1 = 0;
        const double* hcol = u.hp;
        if (gt / 4 < nh) {
            const size_t o_w2 = o_b1 + H, o_b2 = o_w2 + 2 * (size_t)H;
            hcol = ph < o_w2 ? u.hp + 2 * H + (ph - o_b1) : ph < o_b2 ? u.hp + (ph - o_w2) : u.hp + 3 * H + (ph - o_b2);
            const int qn = (u.nhead + 3) / 4;
            q0 = (int)(gt % 4) * qn;
            q1 = min(u.nhead, q0 + qn);
        }
#pragma unroll
        for (int t = 0; t < HQ; ++t) hv[t] = q0 + t < q1 ? __ldg(hcol + (size_t)(q0 + t) * hwd) : 0.0;
        float wh = 0.f;
        if (gt % 4 == 0 && gt / 4 < nh) wh = u.params[ph];
        cluster_wait();
        W16_TR(g.dbg, 5);
        double gs[MAXG][4];
#pragma unroll
        for (int t = 0; t < MAXG; ++t) {
            const int idx = tid + t * NTH;
            gs[t][0] = gs[t][1] = gs[t][2] = gs[t][3] = 0.0;
            if (idx >= n4) continue;
            const uint32_t la = smem_u32(R + (r_lo + idx / B4) * RS + 4 * (idx % B4));
            float pv[S][4];
#pragma unroll
            for (int q = 0; q < S; ++q) {
                uint32_t ra;
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(q));
                asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                             : "=f"(pv[q][0]), "=f"(pv[q][1]), "=f"(pv[q][2]), "=f"(pv[q][3])
                             : "r"(ra)
                             : "memory");
            }
#pragma unroll
            for (int q = 0; q < S; ++q)  // split order (the update kernel's order)
#pragma unroll
                for (int e = 0; e < 4; ++e) gs[t][e] += (double)pv[q][e];
        }
        // the head parameters' sums (their loads were issued before the dump)
        double gh = 0.0;
#pragma unroll
        for (int t = 0; t < HQ; ++t) gh += hv[t];  // (+0.0 past q1: a no-op, gh is never -0)
        for (int q = q0 + HQ; q < q1; ++q) gh += __ldg(hcol + (size_t)q * hwd);  // (nhead > 64)
        gh += __shfl_xor_sync(0xffffffffu, gh, 1);
        gh += __shfl_xor_sync(0xffffffffu, gh, 2);
        cluster_sync();  // every CTA has read the others' partials
        const double loss = sc[0];
        const bool apply = sc[1] < 0.0 && isfinite(loss);  // fit throws before updating (policy.cpp:321-325)
#pragma unroll
        for (int t = 0; t < MAXG; ++t) {
            const int idx = tid + t * NTH;
            const int rl = idx / B4, j = row0 + r_lo + rl;  // output row = parameter row
            if (!apply || idx >= n4 || j >= g.M) continue;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int kl = 4 * (idx % B4) + e, k = col0 + kl;
                if (k >= ncol) continue;
                const float nw = __double2float_rn((double)wold[t][e] - u.lr * gs[t][e]);
                const __nv_bfloat16 b = __float2bfloat16_rn(nw);
                if (w0tile) {  // [X | 1] column: W0 (k < 44), b0 (k == 44)
                    u.params[k < F ? (size_t)j * F + k : o_b0 + j] = nw;
                    if (k < F) u.w0p[(size_t)j * 64 + k] = b;
                } else {
                    u.params[o_w1 + (size_t)j * H + k] = nw;
                    u.w1[(size_t)j * H + k] = b;
                }
            }
        }
        if (apply && gt % 4 == 0 && gt / 4 < nh) u.params[ph] = __double2float_rn((double)wh - u.lr * gh);
        if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && tid == 0 && sc[1] < 0.0) {
            if (isfinite(loss)) *u.epoch_acc += loss * (double)u.nb;
            else *u.diverged = *u.epoch;
        }
    } else {
        OutStage& O = reinterpret_cast<OutStage*>(base)[w];
        for (int c0 = cbeg; c0 < cbeg + CW; c0 += 16) {
            float v[16];
            tmem_ld16(tq + c0, v);
            tmem_ld_wait();
            if (nk == 0) {
#pragma unroll
                for (int i = 0; i < 16; ++i) v[i] = 0.f;
            }
            const int col = col0 + c0;
            if (col >= g.N) break;  // (warp-uniform)
            if constexpr (EPI == W16_EPI_H1) {
                // h1 = relu(acc + b0): row-major (next GEMM's A) + transposed (G4's B)
                float h[16];
#pragma unroll
                for (int i = 0; i < 16; i += 4) {
                    const float4 bb = __ldg(reinterpret_cast<const float4*>(g.bias + col + i));
                    h[i] = fmaxf(v[i] + bb.x, 0.f);
                    h[i + 1] = fmaxf(v[i + 1] + bb.y, 0.f);
                    h[i + 2] = fmaxf(v[i + 2] + bb.z, 0.f);
                    h[i + 3] = fmaxf(v[i + 3] + bb.w, 0.f);
                }
                stage_chunk(O, (c0 - cbeg) >> 4, h, &map_o, &map_ot, col, rw0, lane, true, g.out_t != nullptr);
            } else if constexpr (EPI == W16_EPI_D1T) {
                // d1 = acc [h1 > 0] (mask = stored bf16 H1), transposed (G5's A)
                float h[16];
                const int kq = (c0 - cbeg) >> 4;  // this chunk's two mask words
#pragma unroll
                for (int q2 = 0; q2 < 2; ++q2) {
                    const uint4 mq = kq == 0 ? mk[q2] : kq == 1 ? mk[2 + q2] : kq == 2 ? mk[4 + q2] : mk[6 + q2];
                    const uint32_t wv[4] = {mq.x, mq.y, mq.z, mq.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const __nv_bfloat162 b2 = *reinterpret_cast<const __nv_bfloat162*>(&wv[e]);
                        const int i = 8 * q2 + 2 * e;
                        h[i] = row_ok && __bfloat162float(b2.x) > 0.f ? v[i] : 0.f;
                        h[i + 1] = row_ok && __bfloat162float(b2.y) > 0.f ? v[i + 1] : 0.f;
                    }
                }
                // (one rank: D1 row-major, the fused SGD launch's MN-major A;
                //  data-parallel: D1^T, the split-K G5's K-major A)
                stage_chunk(O, (c0 - cbeg) >> 4, h, &map_o, &map_ot, col, rw0, lane, g.out != nullptr,
                            g.out_t != nullptr);
            } else if (row_ok) {
                // split-K fp32 partial, row-major [M][ldp]
                float4* o = reinterpret_cast<float4*>(g.part + (size_t)blockIdx.z * g.split_stride +
                                                      (size_t)row * g.ldp + col);
#pragma unroll
                for (int q = 0; q < 4; ++q) o[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
            }
        }
        if constexpr (EPI != W16_EPI_PART)
            if (lane == 0) bulk_wait_all();
    }
    fence_before_sync();
    __syncthreads();
    if (w == 0) tmem_dealloc(tacc, TC);
    W16_TR(g.dbg, 3);
}

template __global__ void w16_gemm_kernel<256, 4, W16_EPI_H1>(const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap,
                                                   const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap, W16Args);
template __global__ void w16_gemm_kernel<256, 4, W16_EPI_HEAD>(const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap,
                                                   const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap, W16Args);
template __global__ void w16_gemm_kernel<256, 4, W16_EPI_D1T>(const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap,
                                                   const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap, W16Args);
template __global__ void w16_gemm_kernel<256, 4, W16_EPI_PART>(const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap,
                                                   const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap, W16Args);
template __global__ void w16_gemm_kernel<64, 6, W16_EPI_PART>(const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap,
                                                   const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap, W16Args);
template __global__ void w16_gemm_kernel<128, 6, W16_EPI_SGD>(const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap,
                                                   const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap, W16Args);
template __global__ void w16_gemm_kernel<128, 6, W16_EPI_PART>(const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap,
                                                   const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap, W16Args);

// Xg[r] = bf16(feat[rows[r]]) padded to 64 columns (G1's A); X^T [64][ldt]
// with row 44 = 1 (G5's B: its column 44 of D1^T [X|1] is gb0). A block
// stages 64 rows in shared memory (the gathered 176-byte rows as float4
// loads, all in flight) and writes both layouts with coalesced 16-byte stores.
constexpr int GATHER_ROWS = 64;
__global__ void __launch_bounds__(256) w16_gather_kernel(const float* __restrict__ feat,
                                                         const uint32_t* __restrict__ rows, int nb, int dbg,
                                                         __nv_bfloat16* __restrict__ xg,
                                                         __nv_bfloat16* __restrict__ xt, int ldt) {
    __shared__ __align__(16) __nv_bfloat16 t[GATHER_ROWS][64 + 8];
    W16_TR(dbg, 0);
#ifdef GBX_PHASE_TIMING
    {  // dbg < 0 encodes an untraced step as -(step + 2)
        const int stp = dbg >= 0 ? dbg / 8 : -dbg - 2;
        if (threadIdx.x == 0 && stp >= 0 && stp < 4096) {
            unsigned long long t_;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
            atomicMin(&g_w16_steps[stp], t_);
        }
    }
#endif
    // (no wait here: this step's copy of Xg / X^T is not the one the previous
    //  step's G4+G5 reads, so the gather runs beside it; G1 may launch now —
    //  its own wait covers the gather, which completes only after G4+G5)
    pdl_trigger();
    W16_TR(dbg, 1);
    const int tid = threadIdx.x, r0 = blockIdx.x * GATHER_ROWS;
    const int nr = min(GATHER_ROWS, nb - r0);
    constexpr int NQ = F / 4;  // 11 float4 per row
    float4 v[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const int it = tid + k * 256, r = it / NQ, q = it % NQ;
        v[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (it < GATHER_ROWS * NQ && r < nr)
            v[k] = __ldg(reinterpret_cast<const float4*>(feat + (size_t)rows[r0 + r] * F) + q);
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const int it = tid + k * 256, r = it / NQ, q = it % NQ;
        if (it < GATHER_ROWS * NQ)
            *reinterpret_cast<uint2*>(&t[r][4 * q]) = make_uint2(pack_bf16(v[k].x, v[k].y), pack_bf16(v[k].z, v[k].w));
    }
    // columns 44..63: column 44 = 1 (the ones column of [X | 1]: gb0 in the
    // fused SGD launch; W0p's column 44 is 0, so G1 ignores it), the rest 0
    for (int it = tid; it < GATHER_ROWS * 20; it += 256)
        t[it / 20][F + it % 20] = __float2bfloat16_rn(it % 20 == 0 && it / 20 < nr ? 1.f : 0.f);
    __syncthreads();
    // Xg: 64 rows x 128 B
    for (int it = tid; it < GATHER_ROWS * 8; it += 256) {
        const int r = it >> 3, q = it & 7;
        if (r < nr)
            reinterpret_cast<uint4*>(xg + (size_t)(r0 + r) * 64)[q] = *reinterpret_cast<const uint4*>(&t[r][8 * q]);
    }
    // X^T (data-parallel path only): 64 columns x 64 rows (128 B per column), 8 rows per 16-byte store
    for (int it = tid; xt && it < 64 * 8; it += 256) {
        const int c = it >> 3, rq = (it & 7) * 8;
        if (rq >= nr) continue;
        __nv_bfloat16 e[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
            e[j] = c == F ? (rq + j < nr ? __float2bfloat16_rn(1.f) : __float2bfloat16_rn(0.f)) : t[rq + j][c];
        __nv_bfloat16* dst = xt + (size_t)c * ldt + r0 + rq;
        if (rq + 8 <= nr && ((r0 + rq) & 7) == 0) {
            *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(e);
        } else {
            for (int j = 0; j < 8 && rq + j < nr; ++j) dst[j] = e[j];
        }
    }
    // G1 needs the previous step's update (G4+G5) complete: the gather
    // completes only after it
    pdl_wait();
    W16_TR(dbg, 3);
}

__global__ void to_bf16_kernel(const float* __restrict__ src, size_t n, __nv_bfloat16* __restrict__ dst) {
    const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) dst[t] = __float2bfloat16_rn(src[t]);
}

// BF16 operand copies of the fp32 master weights: W0p [H][64] (K padded),
// W1 [H][H] (G2's B), W1^T [H][H] (G3's B).
__global__ void w16_weights_kernel(const float* __restrict__ params, int H, __nv_bfloat16* __restrict__ w0p,
                                   __nv_bfloat16* __restrict__ w1, __nv_bfloat16* __restrict__ w1t) {
    const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < (size_t)H * 64) {
        const size_t j = t / 64, i = t % 64;
        w0p[t] = __float2bfloat16_rn(i < F ? params[j * F + i] : 0.f);
    }
    if (t >= (size_t)H * H) return;
    const size_t o_w1 = (size_t)H * F + H, k = t / H, j = t % H;
    const __nv_bfloat16 b = __float2bfloat16_rn(params[o_w1 + t]);
    w1[t] = b;
    if (w1t) w1t[j * H + k] = b;
}

// mode 0: reduce + SGD + refreshed bf16 copies (one rank); 1: reduce into the
// flat gradient g_out and the loss sum (before an all-reduce); 2: SGD from g_out.
// Block layout of the update grid: [0, nb2) 1-D over [o_b1, np) (b1, W2, b2:
// the longest sums, over every row tile's head partials, so they start
// first); then [nb2, nb2 + nb0) 1-D over [0, o_w1) (W0, b0); then 32 x 16 W1
// tiles, two parameters per thread (coalesced W1 and W1^T writes through a
// shared-memory transpose). One wave on 148 SMs at H = 512.
__host__ __device__ void w16_update_layout(int H, size_t np, int& nb0, int& nw1, int& nb2) {
    const size_t o_w1 = (size_t)H * F + H, o_b1 = o_w1 + (size_t)H * H;
    nb2 = (int)((np - o_b1 + 255) / 256);
    nb0 = (int)((o_w1 + 255) / 256);
    nw1 = (H / 32) * (H / 16);
}

__global__ void __launch_bounds__(256) w16_update_kernel(W16UpdArgs u, int mode) {
    __shared__ double s_loss;
    __shared__ __nv_bfloat16 s_t[32][17];
    W16_TR(u.dbg, 0);
    pdl_trigger();
    pdl_wait();
    W16_TR(u.dbg, 1);
    const int diverged = *u.diverged;  // (checked after the barrier: its load overlaps the others)
    const int H = u.hidden;
    const size_t o_b0 = (size_t)H * F, o_w1 = o_b0 + H, o_b1 = o_w1 + (size_t)H * H;
    int nb0, nw1, nb2;
    w16_update_layout(H, u.np, nb0, nw1, nb2);
    const int bx = blockIdx.x, tid = threadIdx.x;
    const bool tile = bx >= nb2 + nb0;
    size_t p[2] = {u.np, u.np};
    int tk = 0, tj = 0;
    if (bx < nb2) {
        p[0] = o_b1 + (size_t)bx * 256 + tid;
    } else if (!tile) {
        p[0] = (size_t)(bx - nb2) * 256 + tid;
        if (p[0] >= o_w1) p[0] = u.np;  // (past W0 / b0: idle)
    } else {
        const int t = bx - nb2 - nb0, nt = H / 16;
        tk = t / nt;
        tj = t % nt;
        p[0] = o_w1 + (size_t)(tk * 32 + (tid >> 4)) * H + tj * 16 + (tid & 15);
        p[1] = p[0] + (size_t)16 * H;
    }
    if (mode == 1) {
        if (diverged >= 0) return;
        if (bx == 0 && tid < 32) {
            const double kl = w16_kl_sum(u);
            if (tid == 0) *u.loss_sum = kl;
        }
#pragma unroll
        for (int q = 0; q < 2; ++q)
            if (p[q] < u.np) u.g_out[p[q]] = (float)w16_grad(u, p[q]);
        return;
    }
    // the gradient sums and the old weights are loaded before the loss is
    // known (one round trip for all of them); nothing is written before it is
    double gsum[2] = {0.0, 0.0};
    float wold[2] = {0.f, 0.f};
#pragma unroll
    for (int q = 0; q < 2; ++q)
        if (p[q] < u.np) {
            gsum[q] = mode == 2 ? (double)u.g_out[p[q]] : w16_grad(u, p[q]);
            wold[q] = u.params[p[q]];
        }
    if (tid < 32) {
        const double kl = mode == 2 ? *u.loss_sum : w16_kl_sum(u);
        if (tid == 0) s_loss = kl / (double)u.nb;
    }
    __syncthreads();
    if (diverged >= 0) return;
    W16_TR(u.dbg, 2);
    const double loss = s_loss;
    if (!isfinite(loss)) {  // fit throws before updating (policy.cpp:321-325)
        if (bx == 0 && tid == 0) *u.diverged = *u.epoch;
        return;
    }
    if (bx == 0 && tid == 0) *u.epoch_acc += loss * (double)u.nb;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        if (p[q] >= u.np) continue;
        const float nw = __double2float_rn((double)wold[q] - u.lr * gsum[q]);
        u.params[p[q]] = nw;
        const __nv_bfloat16 b = __float2bfloat16_rn(nw);
        if (p[q] < o_b0) {
            u.w0p[(p[q] / F) * 64 + p[q] % F] = b;
        } else if (tile) {
            u.w1[p[q] - o_w1] = b;
            s_t[(tid >> 4) + 16 * q][tid & 15] = b;
        }
    }
    if (tile && u.w1t) {  // W1^T[j][k] (when a caller keeps one): 32 consecutive k per row of the tile
        __syncthreads();
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int idx = tid + 256 * q, j = idx >> 5, k = idx & 31;
            u.w1t[(size_t)(tj * 16 + j) * H + tk * 32 + k] = s_t[k][j];
        }
    }
    W16_TR(u.dbg, 3);
}

}  // namespace gbxcu

#ifdef GBX_PHASE_TIMING
extern "C" int gbxcu_debug_w16_trace(unsigned long long* out, int reset) {
    if (out && cudaMemcpyFromSymbol(out, gbxcu::g_w16_tr, sizeof(gbxcu::g_w16_tr)) != cudaSuccess) return 3;
    if (reset) {
        static unsigned long long z[64][8][2];
        for (int i = 0; i < 64; ++i)
            for (int j = 0; j < 8; ++j) {
                z[i][j][0] = ~0ull;
                z[i][j][1] = 0;
            }
        if (cudaMemcpyToSymbol(gbxcu::g_w16_tr, z, sizeof(z)) != cudaSuccess) return 3;
    }
    return 0;
}
extern "C" int gbxcu_debug_w16_steps(unsigned long long* out, int reset) {
    if (out && cudaMemcpyFromSymbol(out, gbxcu::g_w16_steps, sizeof(gbxcu::g_w16_steps)) != cudaSuccess) return 3;
    if (reset) {
        static unsigned long long z[4096];
        for (auto& x : z) x = ~0ull;
        if (cudaMemcpyToSymbol(gbxcu::g_w16_steps, z, sizeof(z)) != cudaSuccess) return 3;
    }
    return 0;
}
#endif
