// gbxcu_api.cu — the C ABI declared in include/gbxcu.h.
//
// Host-side orchestration only: argument validation (mirroring the
// reference's ValidationError cases), device buffers, launch configuration,
// the per-epoch shuffle -> train sequence of fit, and the NCCL all-reduce of
// the data-parallel step. All arithmetic on the path runs in the kernels; there
// is no CPU fallback.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/gbxcu.h"
#include "common.cuh"
#include "kernels.h"

using namespace gbxcu;

namespace gbxcu {
template <int BN>
__global__ void tma_gemm_kernel(const __grid_constant__ CUtensorMap map_a,
                                const __grid_constant__ CUtensorMap map_b, GemmArgs g);
}
constexpr int TM_BM_HOST = 128;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CK(call)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return fail(GBXCU_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));     \
    } while (0)

#define CKN(call)                                                                             \
    do {                                                                                      \
        ncclResult_t r_ = (call);                                                             \
        if (r_ != ncclSuccess)                                                                \
            return fail(GBXCU_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_));     \
    } while (0)

#define RET(x)                                         \
    do {                                               \
        int rc_ = (x);                                 \
        if (rc_ != GBXCU_OK) return rc_;               \
    } while (0)

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;  // owns p
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    // grows geometrically once allocated (a table or log that grows a little
    // every call must not pay cudaFree + cudaMalloc, both device-synchronising,
    // every time)
    int ensure(size_t bytes) {
        if (bytes <= cap) return GBXCU_OK;
        const size_t want = std::max<size_t>({bytes, cap ? cap + cap / 2 : 0, 256});
        if (astream) {
            // stream-ordered (pool) allocation on the one stream that uses the
            // buffer: no device-wide synchronisation on growth
            if (p) CK(cudaFreeAsync(p, astream));
            p = nullptr;
            cap = 0;
            CK(cudaMallocAsync(&p, want, astream));
        } else {
            if (p) cudaFree(p);
            p = nullptr;
            cap = 0;
            CK(cudaMalloc(&p, want));
        }
        cap = want;
        return GBXCU_OK;
    }
    cudaStream_t astream = nullptr;  // set: every use of the buffer is on this stream
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
};

}  // namespace

struct gbxcu_ctx {
    int device = 0;
    int num_sms = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;     // gbxcu_fit: epoch-0 shuffle overlapping the H2D
    cudaEvent_t side_ev = nullptr;
    uint64_t launches = 0;
    cudaEvent_t ev[24] = {};                 // fit's per-kernel timing events
    cudaEvent_t eval_ev[3] = {};             // evaluate: before inference | before aggregation | after
    unsigned long long* hres = nullptr;      // pinned host scratch for fit's small results
    double last_shuffle_ms = 0, last_train_ms = 0;
    std::mutex mu;
    // scratch
    DevBuf params, feat, tgt, probs, actions, recheck, counters, flags;
    DevBuf order, order2, partials, red, bar, diverged, epoch_loss, epoch_acc, status;
    DevBuf adam_m, adam_v;  // Adam moments of the fused path (fp64, one per parameter)
    // multi-CTA epoch kernel: exchange regions (counter | LL words | partials)
    // of the peer set. Real peer set: xchg[0] is this rank's (exported),
    // peer_ptr[r] the opened regions of the others. Virtual ranks (single-GPU
    // tests of the peer path): xchg[0..V) all local.
    DevBuf xchg[MAX_PEERS];
    void* peer_ptr[MAX_PEERS] = {};
    int peers = 1, prank = 0;
    uint32_t tag_next = 0;                 // LL tags used so far on the peer set
    unsigned long long ctr_base[MAX_PEERS] = {};  // counter values (identical across a real set)
    DevBuf sh_jp, sh_head, sh_nxt, sh_succ, sh_root, sh_root2, sh_flags;
    DevBuf seg_off, seg_seed, grad, scalar;
    DevBuf s_app_pipe, s_pipe_slot, s_slot_shader, s_slot_frac, s_pipe_wt, s_shader_lat, s_app_f64;
    DevBuf s_actions, s_run_seed, s_rows, s_samples, h_lower, h_count, h_nbins;
    int shuffle_grid = 0;
    int fast_per_sm = 1;
    // wide MLP (C4) working set
    DevBuf w_params, w_grad, w_w1t, w_h1, w_h1t, w_h2, w_d2, w_d2t, w_d1t, w_xt, w_d3, w_kl;
    DevBuf w_part, w_g4, w_g5, w_loss, w_feat, w_tgt, w_probs, w_xg, w_w0p, w_epoch;
    // BF16 path (k_wide16.cu): bf16 activations / operand copies, partials
    DevBuf b_xg, b_xt, b_h1, b_h1t, b_d2, b_d2t, b_d1t, b_w0p, b_w1, b_p4, b_p5, b_hp;
    // CUDA graphs of a wide-MLP epoch's step sequence (one per epoch-permutation
    // buffer), keyed on every pointer and size they bake in
    struct WideGraph {
        std::vector<const void*> key;
        cudaGraphExec_t exec = nullptr;
    } wg[2];
    int wg_next = 0;
    // data parallel
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0;
};

struct gbxcu_dsuite {
    gbxcu_ctx* ctx = nullptr;
    size_t n_apps = 0, n_pipes = 0, n_slots = 0, n_shaders = 0;
    DevBuf app_pipe, pipe_slot, slot_shader, slot_frac, pipe_wt, shader_lat, app_f64, features;
    DevBuf actions, rows, recheck, counters, flags, params, h_lower, h_count, h_nbins;
};

// Device-resident Q-table (row f1): unique keys in StateKey order, two
// optional entries per key (QTable::entries_, proj/include/gbx/qtable.hpp:95-100).
struct gbxcu_qtable {
    gbxcu_ctx* ctx = nullptr;
    double alpha = 0.3, omega = 1.0;
    size_t m = 0;  // states
    DevBuf keys, q, t, cnt, has;
    DevBuf nkeys, nq, nt, ncnt, nhas;  // fold output (swapped in)
    DevBuf bkeys, bact, brew, bnow, init_ids, count;
    DevBuf perm, perm2, digit, digit2, seg_head, key_head, seg_scan, key_scan, seg_start, seg_key;
    DevBuf spread, bad, temp, rn;
    DevBuf flag, row, rowkey, sfeat, stgt, bad_stage;
    DevBuf enc_tab;  // qt_enc_table_kernel output, filled on the first snapshot
    bool enc_ready = false;
};

namespace {

cudaStream_t pick(gbxcu_ctx* c, void* s) { return s ? static_cast<cudaStream_t>(s) : c->stream; }

int setup_kernel_attrs() {
    static std::once_flag once;
    static int rc = GBXCU_OK;
    std::call_once(once, [] {
        auto set = [](const void* fn, size_t bytes) {
            if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) !=
                cudaSuccess) {
                rc = fail(GBXCU_ECUDA, "cudaFuncSetAttribute failed (shared memory opt-in)");
            }
        };
        set((const void*)fwd_fast_kernel, fast_smem_bytes());
        set((const void*)fwd_exact_kernel, exact_smem_bytes());
        set((const void*)fwd_recheck_kernel, recheck_smem_bytes());
        set((const void*)train_epoch_kernel<32>, train_smem_bytes(32));
        set((const void*)train_epoch_kernel<64>, train_smem_bytes(64));
        set((const void*)train_epoch_cluster_kernel, train_cl_smem_bytes());
        set((const void*)train_partial_kernel<32>, train_smem_bytes(32));
        set((const void*)train_partial_kernel<64>, train_smem_bytes(64));
        set((const void*)batch_grad_kernel, train_smem_bytes(64));
        set((const void*)train_epoch_tc_kernel<4, false, false>, train_tc_smem_bytes(4));
        set((const void*)train_epoch_tc_kernel<7, false, false>, train_tc_smem_bytes(7));
        set((const void*)train_epoch_tc_kernel<4, true, false>, train_tc_smem_bytes(4));
        set((const void*)train_epoch_tc_kernel<7, true, false>, train_tc_smem_bytes(7));
        set((const void*)train_epoch_tc_kernel<4, false, true>, train_tc_smem_bytes(4));
        set((const void*)train_epoch_tc_kernel<7, false, true>, train_tc_smem_bytes(7));
        set((const void*)train_epoch_tc_kernel<4, true, true>, train_tc_smem_bytes(4));
        set((const void*)train_epoch_tc_kernel<7, true, true>, train_tc_smem_bytes(7));
        set((const void*)train_partial_tc_kernel<4>, train_tc_smem_bytes(4));
        set((const void*)train_partial_tc_kernel<7>, train_tc_smem_bytes(7));
        set((const void*)tc_gemm_kernel, gemm_smem_bytes());
        set((const void*)wide_head_kernel, sizeof(float) * 32 * (1024 + 1));
        set((const void*)tma_gemm_kernel<64>, tma_gemm_smem_bytes<64>());
        set((const void*)w16_gemm_kernel<256, 4, W16_EPI_H1>, w16_gemm_smem_bytes<256, 4>());
        set((const void*)w16_gemm_kernel<256, 4, W16_EPI_HEAD>, w16_gemm_smem_bytes<256, 4>());
        set((const void*)w16_gemm_kernel<256, 4, W16_EPI_D1T>, w16_gemm_smem_bytes<256, 4>());
        set((const void*)w16_gemm_kernel<256, 4, W16_EPI_PART>, w16_gemm_smem_bytes<256, 4>());
        set((const void*)w16_gemm_kernel<64, 6, W16_EPI_PART>, w16_gemm_smem_bytes<64, 6>());
        set((const void*)w16_gemm_kernel<128, 6, W16_EPI_PART>, w16_gemm_smem_bytes<128, 6>());
        set((const void*)w16_gemm_kernel<128, 6, W16_EPI_SGD>, w16_gemm_smem_bytes<128, 6>());
        set((const void*)tma_gemm_kernel<128>, tma_gemm_smem_bytes<128>());
        set((const void*)tma_gemm_kernel<256>, tma_gemm_smem_bytes<256>());
    });
    return rc;
}

int check_launch(gbxcu_ctx* c, const char* what) {
    c->launches++;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(GBXCU_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
    return GBXCU_OK;
}

// ------------------------------------------------------------- inference
int run_forward(gbxcu_ctx* c, const float* d_params, const float* d_feat, size_t n,
                double* d_probs, uint8_t* d_actions, int mode, const uint64_t* d_seg_off,
                size_t nseg, const uint64_t* d_seg_seed, double eps, cudaStream_t st,
                DevBuf& recheck, DevBuf& counters, DevBuf& flags, int extra_bits = 0) {
    if (n == 0) return GBXCU_OK;
    if (n > 0xFFFFFFFFull) return fail(GBXCU_EINVAL, "batch too large (> 2^32 states)");
    const int bits = (d_probs ? FWD_PROBS : 0) | (d_actions ? FWD_ACTIONS : 0) |
                     (d_seg_off ? FWD_COLLECT : 0) | extra_bits;
    RET(counters.ensure(16));
    RET(flags.ensure(16));
    CK(cudaMemsetAsync(counters.p, 0, 16, st));
    CK(cudaMemsetAsync(flags.p, 0, 16, st));
    if (mode == GBXCU_FWD_FAST) {
        RET(recheck.ensure(n * sizeof(uint32_t)));
        const size_t warps = (n + 63) / 64;  // 64 states per warp pass
        const size_t blocks_needed = (warps + FWD_BLOCK / 32 - 1) / (FWD_BLOCK / 32);
        const int grid = (int)std::min<size_t>(blocks_needed, (size_t)c->num_sms * c->fast_per_sm);
        fwd_fast_kernel<<<grid, FWD_BLOCK, fast_smem_bytes(), st>>>(
            d_params, d_feat, n, d_probs, d_actions, d_seg_off, nseg, d_seg_seed, eps,
            recheck.as<uint32_t>(), counters.as<unsigned int>(), flags.as<unsigned int>(), bits);
        RET(check_launch(c, "fwd_fast_kernel"));
        // the list length stays on the device: a fixed grid, idle blocks exit at once
        fwd_recheck_kernel<<<c->num_sms * 3, RECHECK_BLOCK, recheck_smem_bytes(), st>>>(
            d_params, d_feat, recheck.as<uint32_t>(), counters.as<unsigned int>(), d_probs,
            d_actions, d_seg_off, nseg, d_seg_seed, eps, bits);
        RET(check_launch(c, "fwd_recheck_kernel"));
    } else {
        // one resident wave (2 CTAs/SM at the kernel's register count), grid-stride:
        // each CTA builds its fp64 weight copy once
        const size_t blocks_needed = (n + EXACT_BLOCK - 1) / EXACT_BLOCK;
        const int grid = (int)std::min<size_t>(blocks_needed, (size_t)c->num_sms * 2);
        fwd_exact_kernel<<<grid, EXACT_BLOCK, exact_smem_bytes(), st>>>(
            d_params, d_feat, n, nullptr, nullptr, d_probs, d_actions, d_seg_off, nseg,
            d_seg_seed, eps, flags.as<unsigned int>(), bits);
        RET(check_launch(c, "fwd_exact_kernel"));
    }
    return GBXCU_OK;
}

// aggregation: AGG_APPS apps per warp, one resident wave, grid-stride beyond it
int launch_aggregate(gbxcu_ctx* c, const AggArgs& a, cudaStream_t st) {
    const size_t per_cta = (size_t)(AGG_BLOCK / 32) * AGG_APPS;
    const int grid = (int)std::max<size_t>(1, std::min<size_t>((a.n_apps + per_cta - 1) / per_cta,
                                                               (size_t)c->num_sms * AGG_MINB));
    aggregate_kernel<AGG_APPS, AGG_MINB><<<grid, AGG_BLOCK, 0, st>>>(a);
    return check_launch(c, "aggregate_kernel");
}

int check_flags(DevBuf& flags, cudaStream_t st) {
    unsigned int f = 0;
    CK(cudaMemcpyAsync(&f, flags.p, sizeof(f), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (f & 1u) return fail(GBXCU_ENONFINITE, "non-finite feature in shader state");
    return GBXCU_OK;
}

// ------------------------------------------------------------------- fit
int validate_cfg(const gbxcu_train_cfg* cfg, size_t n) {
    if (!cfg) return fail(GBXCU_EINVAL, "null train config");
    if (!(cfg->learning_rate > 0.0)) return fail(GBXCU_EINVAL, "learning rate must be positive");
    if (cfg->epochs < 1) return fail(GBXCU_EINVAL, "epochs must be >= 1");
    if (cfg->batch_size < 1) return fail(GBXCU_EINVAL, "batch size must be >= 1");
    if (n == 0) return fail(GBXCU_EINVAL, "fit requires a non-empty dataset");
    if (n > 0x7FFFFFFFull) return fail(GBXCU_EINVAL, "dataset too large (> 2^31 records)");
    if (cfg->loss_mode != GBXCU_LOSS_KL && cfg->loss_mode != GBXCU_LOSS_TD)
        return fail(GBXCU_EINVAL, "unknown loss mode");
    if (cfg->optimizer != GBXCU_OPT_SGD && cfg->optimizer != GBXCU_OPT_ADAM)
        return fail(GBXCU_EINVAL, "unknown optimizer");
    if (cfg->optimizer == GBXCU_OPT_ADAM) {
        const double b1 = cfg->adam_beta1, b2 = cfg->adam_beta2, ep = cfg->adam_eps;
        if (!(b1 >= 0.0 && b1 < 1.0) || !(b2 >= 0.0 && b2 < 1.0) || !(ep >= 0.0))
            return fail(GBXCU_EINVAL, "Adam needs 0 <= beta < 1 and eps >= 0 (0 = default)");
    }
    return GBXCU_OK;
}

// CTAs per step and records per tile: spread each rank's share of the batch
// over up to one CTA per SM in tiles of 32 records; switch to 64-record
// tiles once every SM already has more than 32 records.
void train_grid(gbxcu_ctx* c, const gbxcu_train_cfg* cfg, size_t n, int nranks, int& G, int& tb,
                int sm_share = 1) {
    const size_t b = std::min<size_t>((size_t)cfg->batch_size, n);
    const size_t per_rank = (b + nranks - 1) / nranks;
    G = (int)std::min<size_t>((per_rank + 31) / 32, (size_t)(c->num_sms / sm_share));
    if (cfg->max_ctas > 0) G = std::min(G, cfg->max_ctas);
    G = std::max(G, 1);
    const size_t per_cta = (per_rank + G - 1) / G;
    tb = per_cta <= 32 ? 32 : 64;
}

// One epoch's Fisher-Yates pass: order -> order2, then the two are swapped.
int shuffle_epoch(gbxcu_ctx* c, size_t n, uint64_t seed, int epoch, cudaStream_t st) {
    if (n < 2) return GBXCU_OK;
    ShuffleArgs s{};
    s.in = c->order.as<uint32_t>();
    s.out = c->order2.as<uint32_t>();
    s.n = (uint32_t)n;
    s.seed_e = derive_seed3(seed, 0x5F17u, (uint64_t)epoch);
    s.jp = c->sh_jp.as<uint32_t>();
    s.head = c->sh_head.as<uint32_t>();
    s.nxt = c->sh_nxt.as<uint32_t>();
    s.succ = c->sh_succ.as<uint32_t>();
    s.root = c->sh_root.as<uint32_t>();
    s.root2 = c->sh_root2.as<uint32_t>();
    s.flags = c->sh_flags.as<unsigned int>();
    s.fg0 = c->sh_flags.as<uint32_t>() + 64;
    s.bar = c->sh_flags.as<unsigned int>() + 72;
    s.diverged = c->diverged.as<int>();
    CK(cudaMemsetAsync(c->sh_flags.p, 0, 80 * sizeof(uint32_t), st));
    void* args[] = {&s};
    CK(cudaLaunchCooperativeKernel((const void*)shuffle_epoch_kernel, c->shuffle_grid, SHUF_BLOCK,
                                   args, 0, st));
    std::swap(c->order.p, c->order2.p);
    std::swap(c->order.cap, c->order2.cap);
    return check_launch(c, "shuffle_epoch_kernel");
}

int prepare_order(gbxcu_ctx* c, size_t n, cudaStream_t st) {
    for (DevBuf* b : {&c->order, &c->order2, &c->sh_jp, &c->sh_head, &c->sh_nxt, &c->sh_succ,
                      &c->sh_root, &c->sh_root2})
        RET(b->ensure(n * 4));
    RET(c->sh_flags.ensure(80 * sizeof(uint32_t)));
    // epoch e of every call reads the same buffer (shuffle_epoch ping-pongs
    // order / order2): graphs captured over an epoch's steps stay valid
    if (c->order.p > c->order2.p) {
        std::swap(c->order.p, c->order2.p);
        std::swap(c->order.cap, c->order2.cap);
    }
    RET(c->bar.ensure(16));
    RET(c->diverged.ensure(16));
    CK(cudaMemsetAsync(c->diverged.p, 0xFF, 16, st));
    iota_kernel<<<std::max(1, std::min<int>((int)((n + 255) / 256), c->num_sms * 8)), 256, 0, st>>>(
        c->order.as<uint32_t>(), n);
    return check_launch(c, "iota_kernel");
}

// Exchange region layout (one per rank; 256-B aligned sections):
//   [u64 arrival counter | pad][NP u64 LL parameter words]
//   [2 x (NP + 1) u64 LL per-GPU sums (peer sets)][G x PSTR f64 partial rows]
constexpr size_t xchg_align(size_t b) { return (b + 255) / 256 * 256; }
constexpr size_t XCHG_LL_OFF = 256;
constexpr size_t XCHG_GP_OFF = XCHG_LL_OFF + xchg_align(NP * 8);
constexpr size_t XCHG_PART_OFF = XCHG_GP_OFF + xchg_align(2 * (NP + 1) * 8);
size_t xchg_bytes(int g) { return XCHG_PART_OFF + (size_t)g * PSTR * sizeof(double); }

int ensure_xchg(gbxcu_ctx* c, int slot, int g, cudaStream_t st) {
    if (c->xchg[slot].cap >= xchg_bytes(g)) return GBXCU_OK;
    CK(cudaStreamSynchronize(st));
    RET(c->xchg[slot].ensure(xchg_bytes(g)));
    CK(cudaMemsetAsync(c->xchg[slot].p, 0, xchg_bytes(g), st));
    c->ctr_base[slot] = 0;
    return GBXCU_OK;
}

void bind_region(TrainArgs& a, int r, void* base) {
    auto* b = static_cast<unsigned char*>(base);
    a.ctr[r] = reinterpret_cast<unsigned long long*>(b);
    a.llp[r] = reinterpret_cast<unsigned long long*>(b + XCHG_LL_OFF);
    a.gp[r] = reinterpret_cast<unsigned long long*>(b + XCHG_GP_OFF);
    a.part[r] = reinterpret_cast<double*>(b + XCHG_PART_OFF);
}

int fit_device(gbxcu_ctx* c, float* d_params, const float* d_feat, const double* d_tgt, size_t n,
               const gbxcu_train_cfg* cfg, double* epoch_loss_out, int* diverged_epoch,
               cudaStream_t st, bool pre_shuffled = false) {
    RET(validate_cfg(cfg, n));
    RET(setup_kernel_attrs());
    // pre_shuffled: the caller already ran prepare_order + epoch 0's shuffle
    // (gbxcu_fit overlaps them with the host-to-device copies)
    if (!pre_shuffled) RET(prepare_order(c, n, st));
    RET(c->epoch_loss.ensure(sizeof(double) * cfg->epochs));
    RET(c->epoch_acc.ensure(16));
    if (c->peers < 0) return fail(GBXCU_EINVAL, "peer set timed out earlier; re-attach it");
    // Peer set of the fused multi-CTA path: a real one (gbxcu_peer_attach: one
    // process per GPU), or cfg->virtual_ranks virtual ranks inside one launch
    // (single-GPU tests of the same kernel path).
    if (cfg->virtual_ranks > 1 && (c->peers > 1 || c->comm))
        return fail(GBXCU_EINVAL, "virtual ranks need a context without peers or communicator");
    const int vranks = c->peers > 1 ? 1 : std::max(1, cfg->virtual_ranks);
    const int eff_ranks = vranks > 1 ? vranks : c->nranks;
    int G = 1, tb = 32;
    train_grid(c, cfg, n, eff_ranks, G, tb, vranks);
    RET(c->partials.ensure(sizeof(double) * (size_t)G * PSTR));
    RET(c->red.ensure(sizeof(double) * (NP + 1)));
    RET(c->status.ensure(16));
    CK(cudaMemsetAsync(c->status.p, 0, 16, st));
    // multi-CTA steps: tensor-core kernel, tiles of 32 (MT 4) or 56 (MT 7) records
    const size_t per_cta = ((std::min<size_t>((size_t)cfg->batch_size, n) + eff_ranks - 1) /
                                eff_ranks + G - 1) / G;
    const int mt = per_cta <= 32 ? 4 : 7;
    // the variants (TD loss, Adam) run on the fused tensor-core kernel at every
    // grid size; the bit-exact 1-CTA kernel and the NCCL path are the reference's
    const bool variant = cfg->loss_mode != GBXCU_LOSS_KL || cfg->optimizer != GBXCU_OPT_SGD;
    if (variant && c->comm)
        return fail(GBXCU_EINVAL, "TD loss / Adam need the fused path (no NCCL communicator)");
    const bool fused = !c->comm && (G > 1 || variant);
    if (vranks > MAX_PEERS || vranks * G > c->num_sms)
        return fail(GBXCU_EINVAL, "virtual ranks x CTAs exceed the GPU");
    if (vranks > 1 && G == 1) return fail(GBXCU_EINVAL, "virtual ranks need multi-CTA steps");
    if (c->peers > 1 && c->comm) return fail(GBXCU_EINVAL, "peer set and NCCL communicator both attached");
    if (c->peers > 1 && G == 1) return fail(GBXCU_EINVAL, "peer set needs multi-CTA steps (batch > 32 per rank)");
    if (c->peers > 1 && c->xchg[0].cap < xchg_bytes(G))
        return fail(GBXCU_EINVAL, "peer exchange region too small for this grid");
    if (c->peers == 1) {
        // local peer set (this GPU alone, or virtual ranks): this process owns
        // every region, so the arrival counters restart at 0 each fit. LL tags
        // stay monotonic over the context's life (stale words never match).
        for (int r = 0; r < vranks; ++r) {
            RET(ensure_xchg(c, r, G, st));
            CK(cudaMemsetAsync(c->xchg[r].p, 0, sizeof(unsigned long long), st));
            c->ctr_base[r] = 0;
        }
    }
    TrainArgs a{};
    a.feat = d_feat;
    a.tgt = d_tgt;
    a.order = c->order.as<uint32_t>();
    a.params = d_params;
    a.partials = c->partials.as<double>();
    a.bar = c->bar.as<unsigned int>() + 2;  // separate from the shuffle's counter
    a.diverged_epoch = c->diverged.as<int>();
    a.epoch_loss = c->epoch_loss.as<double>();
    a.n = n;
    a.batch = cfg->batch_size;
    a.lr = cfg->learning_rate;
    a.rank = c->rank;
    a.nranks = c->nranks;
    a.status = c->status.as<int>();
    const int R = c->peers > 1 ? c->peers : vranks;
    a.peers = R;
    a.prank = c->peers > 1 ? c->prank : 0;
    a.pvirt = c->peers > 1 ? 0 : (vranks > 1 ? 1 : 0);
    for (int r = 0; r < R; ++r)
        bind_region(a, r, c->peers > 1 ? (r == c->prank ? c->xchg[0].p : c->peer_ptr[r]) : c->xchg[r].p);
    if (a.pvirt) {  // each virtual rank trains its slice of every global batch
        a.nranks = R;
        a.rank = 0;
    }
    const int GG = R * G;
    const long n_steps = (long)((n + cfg->batch_size - 1) / cfg->batch_size);
    a.loss_mode = cfg->loss_mode;
    a.optimizer = cfg->optimizer;
    a.beta1 = cfg->adam_beta1 > 0.0 ? cfg->adam_beta1 : 0.9;
    a.beta2 = cfg->adam_beta2 > 0.0 ? cfg->adam_beta2 : 0.999;
    a.adam_eps = cfg->adam_eps > 0.0 ? cfg->adam_eps : 1e-8;
    if (cfg->optimizer == GBXCU_OPT_ADAM) {  // fresh moments per fit (t counts the fit's steps)
        RET(c->adam_m.ensure(sizeof(double) * NP));
        RET(c->adam_v.ensure(sizeof(double) * NP));
        CK(cudaMemsetAsync(c->adam_m.p, 0, sizeof(double) * NP, st));
        CK(cudaMemsetAsync(c->adam_v.p, 0, sizeof(double) * NP, st));
        a.adam_m = c->adam_m.as<double>();
        a.adam_v = c->adam_v.as<double>();
    }

    const bool timed = cfg->epochs <= 8;  // per-kernel event timing (bench / profiling)
    for (int e = 0; e < cfg->epochs; ++e) {
        if (timed) CK(cudaEventRecord(c->ev[2 * e % 16], st));
        if (!(pre_shuffled && e == 0)) RET(shuffle_epoch(c, n, cfg->seed, e, st));
        a.order = c->order.as<uint32_t>();  // the pass output (buffers ping-pong)
        a.epoch = e;
        a.tag_base = c->tag_next + (unsigned int)((long)e * n_steps);
        // each rank's counter counts its own CTAs' arrivals (G per step)
        a.ctr_base = c->ctr_base[0] + (unsigned long long)e * n_steps * G;
        a.step0 = (unsigned)((long)e * n_steps);
        if (!c->comm) {
            void* args[] = {&a};
            if (timed) CK(cudaEventRecord(c->ev[(2 * e + 1) % 16], st));
            if (!fused) {
                // 1-CTA steps: the bit-exact fp64 kernel (reference summation
                // order); batches <= 32 on one rank spread each step over a
                // cluster of CTAs (same chains, same order)
                static const bool one_cta = getenv("GBX_TRAIN32_1CTA") != nullptr;  // (A/B timing)
                if (tb == 32 && c->nranks == 1 && !one_cta) {
                    CK(cudaLaunchKernel((const void*)train_epoch_cluster_kernel, TRAIN_CLUSTER, TRAIN_BLOCK,
                                        args, train_cl_smem_bytes(), st));
                } else {
                    const void* fn = tb == 32 ? (const void*)train_epoch_kernel<32>
                                              : (const void*)train_epoch_kernel<64>;
                    CK(cudaLaunchKernel(fn, 1, TRAIN_BLOCK, args, train_smem_bytes(tb), st));
                }
            } else {
                // system-scope exchange only across GPUs (a real peer set)
                const bool sys = c->peers > 1;
                // variants (TD loss / Adam) in their own instantiations: the
                // reference's KL + SGD kernels carry no runtime branches for them
                const void* fns[2][2][2] = {
                    {{(const void*)train_epoch_tc_kernel<4, false, false>,
                      (const void*)train_epoch_tc_kernel<4, false, true>},
                     {(const void*)train_epoch_tc_kernel<4, true, false>,
                      (const void*)train_epoch_tc_kernel<4, true, true>}},
                    {{(const void*)train_epoch_tc_kernel<7, false, false>,
                      (const void*)train_epoch_tc_kernel<7, false, true>},
                     {(const void*)train_epoch_tc_kernel<7, true, false>,
                      (const void*)train_epoch_tc_kernel<7, true, true>}}};
                const void* fn = fns[mt == 4 ? 0 : 1][sys ? 1 : 0][variant ? 1 : 0];
                CK(cudaLaunchCooperativeKernel(fn, a.pvirt ? GG : G, TRAIN_BLOCK, args,
                                               train_tc_smem_bytes(mt), st));
            }
            RET(check_launch(c, "train_epoch_kernel"));
            if (timed) CK(cudaEventRecord(c->ev[16 + e % 8], st));
        } else {
            CK(cudaMemsetAsync(c->epoch_acc.p, 0, sizeof(double), st));
            for (long s = 0; s < n_steps; ++s) {
                const size_t start = (size_t)s * cfg->batch_size;
                const size_t nb = std::min(n, start + (size_t)cfg->batch_size) - start;
                if (G == 1 && tb == 32)
                    train_partial_kernel<32><<<G, TRAIN_BLOCK, train_smem_bytes(32), st>>>(a, s);
                else if (G == 1)
                    train_partial_kernel<64><<<G, TRAIN_BLOCK, train_smem_bytes(64), st>>>(a, s);
                else if (mt == 4)
                    train_partial_tc_kernel<4><<<G, TRAIN_BLOCK, train_tc_smem_bytes(4), st>>>(a, s);
                else
                    train_partial_tc_kernel<7><<<G, TRAIN_BLOCK, train_tc_smem_bytes(7), st>>>(a, s);
                RET(check_launch(c, "train_partial_kernel"));
                reduce_partials_kernel<<<(NP + 1 + 7) / 8, 256, 0, st>>>(
                    c->partials.as<double>(), G, c->red.as<double>(), c->diverged.as<int>());
                RET(check_launch(c, "reduce_partials_kernel"));
                CKN(ncclAllReduce(c->red.p, c->red.p, NP + 1, ncclFloat64, ncclSum, c->comm, st));
                apply_update_kernel<<<(NP + 255) / 256, 256, 0, st>>>(
                    d_params, c->red.as<double>(), cfg->learning_rate, nb, e,
                    c->diverged.as<int>(), c->epoch_acc.as<double>());
                RET(check_launch(c, "apply_update_kernel"));
            }
            finish_epoch_kernel<<<1, 1, 0, st>>>(c->epoch_acc.as<double>(), n, e,
                                                  c->diverged.as<int>(), c->epoch_loss.as<double>());
            RET(check_launch(c, "finish_epoch_kernel"));
        }
    }
    // small results into pinned scratch: truly asynchronous copies, one sync
    // (pageable destinations make each copy a blocking round trip)
    unsigned long long local[2 + MAX_PEERS] = {};
    unsigned long long* hr = c->hres ? c->hres : local;
    int* hdv = reinterpret_cast<int*>(hr);  // hr[0] = {diverged, status}
    CK(cudaMemcpyAsync(hdv, c->diverged.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hdv + 1, c->status.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    const bool used_tc = fused;
    const int n_ctr = used_tc ? (c->peers > 1 ? 1 : vranks) : 0;
    for (int r = 0; r < n_ctr; ++r)  // resynchronise the monotonic counters (divergence stops early)
        CK(cudaMemcpyAsync(hr + 1 + r, c->xchg[r].p, sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, st));
    const bool loss_via_scratch = epoch_loss_out && c->hres && cfg->epochs <= 48;
    if (epoch_loss_out)
        CK(cudaMemcpyAsync(loss_via_scratch ? static_cast<void*>(hr + 16) : epoch_loss_out,
                           c->epoch_loss.p, sizeof(double) * cfg->epochs, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (loss_via_scratch) std::memcpy(epoch_loss_out, hr + 16, sizeof(double) * cfg->epochs);
    const int dv = hdv[0], wd = hdv[1];
    for (int r = 0; r < n_ctr; ++r) c->ctr_base[r] = hr[1 + r];
    c->last_shuffle_ms = c->last_train_ms = 0.0;
    if (timed && !c->comm) {
        for (int e = 0; e < cfg->epochs; ++e) {
            float a_ms = 0.f, b_ms = 0.f;
            cudaEventElapsedTime(&a_ms, c->ev[2 * e % 16], c->ev[(2 * e + 1) % 16]);
            cudaEventElapsedTime(&b_ms, c->ev[(2 * e + 1) % 16], c->ev[16 + e % 8]);
            c->last_shuffle_ms += a_ms;
            c->last_train_ms += b_ms;
        }
    }
    if (used_tc) c->tag_next += (uint32_t)((long)cfg->epochs * n_steps);
    if (wd != 0) {
        c->peers = c->peers > 1 ? -c->peers : c->peers;  // the set is unusable until re-attached
        return fail(GBXCU_ECUDA, "peer synchronisation timed out (a rank stopped responding)");
    }
    if (diverged_epoch) *diverged_epoch = dv;
    if (dv >= 0)
        return fail(GBXCU_EDIVERGED,
                    "training loss became non-finite at epoch " + std::to_string(dv));
    return GBXCU_OK;
}

// Host or device source (unified addressing decides the copy direction).
template <typename T>
int upload(DevBuf& b, const T* src, size_t count, cudaStream_t st) {
    RET(b.ensure(sizeof(T) * count));
    if (count) CK(cudaMemcpyAsync(b.p, src, sizeof(T) * count, cudaMemcpyDefault, st));
    return GBXCU_OK;
}

int suite_args(const gbxcu_suite* s) {
    if (!s) return fail(GBXCU_EINVAL, "null suite");
    if (s->n_apps && (!s->app_pipe_off || !s->pipe_slot_off || !s->app_f64))
        return fail(GBXCU_EINVAL, "suite arrays missing");
    return GBXCU_OK;
}

}  // namespace

// =========================================================================
extern "C" {

int gbxcu_abi_version(void) { return GBXCU_ABI_VERSION; }
const char* gbxcu_last_error(void) { return g_err.c_str(); }

int gbxcu_create(int device, gbxcu_ctx** out) {
    if (!out) return fail(GBXCU_EINVAL, "null output pointer");
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        return fail(GBXCU_ECUDA, std::string("no CUDA device available: ") +
                                     (e == cudaSuccess ? "0 devices" : cudaGetErrorString(e)));
    if (device < 0 || device >= count) return fail(GBXCU_EINVAL, "device index out of range");
    CK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        return fail(GBXCU_ECUDA, std::string("gbxcu is built for sm_100a (B200); device is ") +
                                     prop.name);
    auto* c = new gbxcu_ctx;
    c->device = device;
    c->num_sms = prop.multiProcessorCount;
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->side_ev, cudaEventDisableTiming) != cudaSuccess) {
        delete c;
        return fail(GBXCU_ECUDA, "cudaStreamCreate failed");
    }
    int rc = setup_kernel_attrs();
    if (rc != GBXCU_OK) {
        delete c;
        return rc;
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, shuffle_epoch_kernel, SHUF_BLOCK, 0);
    c->shuffle_grid = std::max(1, std::min(per_sm, 4)) * c->num_sms;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fwd_fast_kernel, FWD_BLOCK,
                                                  fast_smem_bytes());
    c->fast_per_sm = std::max(1, per_sm);
    for (auto& e : c->ev) cudaEventCreate(&e);
    for (auto& e : c->eval_ev) cudaEventCreate(&e);
    {  // keep freed stream-ordered allocations in the pool (reused, not returned)
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t keep = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
    }
    if (cudaHostAlloc(reinterpret_cast<void**>(&c->hres), 64 * sizeof(unsigned long long),
                      cudaHostAllocDefault) != cudaSuccess)
        c->hres = nullptr;  // fall back to pageable copies (slower, same results)
    *out = c;
    return GBXCU_OK;
}

void gbxcu_destroy(gbxcu_ctx* c) {
    if (!c) return;
    if (c->comm) ncclCommDestroy(c->comm);
    for (auto& p : c->peer_ptr)
        if (p) cudaIpcCloseMemHandle(p);
    for (auto& e : c->eval_ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : c->ev)
        if (e) cudaEventDestroy(e);
    for (auto& g : c->wg)
        if (g.exec) cudaGraphExecDestroy(g.exec);
    if (c->stream) cudaStreamDestroy(c->stream);
    if (c->side) cudaStreamDestroy(c->side);
    if (c->side_ev) cudaEventDestroy(c->side_ev);
    if (c->hres) cudaFreeHost(c->hres);
    delete c;
}

void* gbxcu_stream(gbxcu_ctx* c) { return c ? (void*)c->stream : nullptr; }
uint64_t gbxcu_launch_count(const gbxcu_ctx* c) { return c ? c->launches : 0; }

int gbxcu_last_fit_timing(const gbxcu_ctx* c, double* shuffle_ms, double* train_kernel_ms) {
    if (!c) return fail(GBXCU_EINVAL, "null context");
    if (shuffle_ms) *shuffle_ms = c->last_shuffle_ms;
    if (train_kernel_ms) *train_kernel_ms = c->last_train_ms;
    return GBXCU_OK;
}

int gbxcu_last_eval_timing(gbxcu_ctx* c, double* infer_ms, double* aggregate_ms) {
    if (!c) return fail(GBXCU_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    CK(cudaEventSynchronize(c->eval_ev[2]));
    float a = 0.f, b = 0.f;
    CK(cudaEventElapsedTime(&a, c->eval_ev[0], c->eval_ev[1]));
    CK(cudaEventElapsedTime(&b, c->eval_ev[1], c->eval_ev[2]));
    if (infer_ms) *infer_ms = a;
    if (aggregate_ms) *aggregate_ms = b;
    return GBXCU_OK;
}

int gbxcu_last_recheck_count(gbxcu_ctx* c, uint64_t* count) {
    if (!c || !count) return fail(GBXCU_EINVAL, "null argument");
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    unsigned int v = 0;
    if (c->counters.p) {
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(&v, c->counters.p, sizeof(v), cudaMemcpyDeviceToHost));
    }
    *count = v;
    return GBXCU_OK;
}

int gbxcu_policy_init(gbxcu_ctx* c, uint64_t seed, float* params_out) {
    if (!c || !params_out) return fail(GBXCU_EINVAL, "null argument");
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    RET(c->params.ensure(sizeof(float) * NP));
    policy_init_kernel<<<(NP + 255) / 256, 256, 0, c->stream>>>(seed, c->params.as<float>());
    RET(check_launch(c, "policy_init_kernel"));
    CK(cudaMemcpyAsync(params_out, c->params.p, sizeof(float) * NP, cudaMemcpyDeviceToHost,
                       c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return GBXCU_OK;
}

int gbxcu_forward(gbxcu_ctx* c, const float* params, const float* feat, size_t n, double* probs,
                  uint8_t* actions, int mode) {
    if (!c || !params || (n && !feat)) return fail(GBXCU_EINVAL, "null argument");
    if (mode != GBXCU_FWD_EXACT && mode != GBXCU_FWD_FAST) return fail(GBXCU_EINVAL, "bad mode");
    if (n == 0) return GBXCU_OK;
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    RET(upload(c->params, params, NP, st));
    RET(upload(c->feat, feat, n * F, st));
    RET(c->probs.ensure(probs ? n * 16 : 16));
    RET(c->actions.ensure(actions ? n : 16));
    RET(run_forward(c, c->params.as<float>(), c->feat.as<float>(), n,
                    probs ? c->probs.as<double>() : nullptr,
                    actions ? c->actions.as<uint8_t>() : nullptr, mode, nullptr, 0, nullptr, 0.0,
                    st, c->recheck, c->counters, c->flags));
    RET(check_flags(c->flags, st));
    if (probs) CK(cudaMemcpyAsync(probs, c->probs.p, n * 16, cudaMemcpyDeviceToHost, st));
    if (actions) CK(cudaMemcpyAsync(actions, c->actions.p, n, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return GBXCU_OK;
}

int gbxcu_forward_dev(gbxcu_ctx* c, const float* d_params, const float* d_feat, size_t n,
                      double* d_probs, uint8_t* d_actions, int mode, void* stream) {
    if (!c || !d_params || (n && !d_feat)) return fail(GBXCU_EINVAL, "null argument");
    if (mode != GBXCU_FWD_EXACT && mode != GBXCU_FWD_FAST) return fail(GBXCU_EINVAL, "bad mode");
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    return run_forward(c, d_params, d_feat, n, d_probs, d_actions, mode, nullptr, 0, nullptr, 0.0,
                       pick(c, stream), c->recheck, c->counters, c->flags);
}

int gbxcu_collect(gbxcu_ctx* c, const float* params, const float* feat, const uint64_t* seg_off,
                  size_t nseg, const uint64_t* seg_seed, double eps, uint8_t* actions) {
    if (!c || !params || !seg_off || !seg_seed || !actions) return fail(GBXCU_EINVAL, "null argument");
    const size_t n = nseg ? seg_off[nseg] : 0;
    if (n == 0) return GBXCU_OK;
    if (seg_off[0] != 0) return fail(GBXCU_EINVAL, "segment offsets must start at 0");
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    RET(upload(c->params, params, NP, st));
    RET(upload(c->feat, feat, n * F, st));
    RET(upload(c->seg_off, seg_off, nseg + 1, st));
    RET(upload(c->seg_seed, seg_seed, nseg, st));
    RET(c->actions.ensure(n));
    RET(run_forward(c, c->params.as<float>(), c->feat.as<float>(), n, nullptr,
                    c->actions.as<uint8_t>(), GBXCU_FWD_FAST, c->seg_off.as<uint64_t>(), nseg,
                    c->seg_seed.as<uint64_t>(), eps, st, c->recheck, c->counters, c->flags));
    RET(check_flags(c->flags, st));
    CK(cudaMemcpyAsync(actions, c->actions.p, n, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return GBXCU_OK;
}

int gbxcu_forward_batch(gbxcu_ctx* c, const float* params, const float* feat, size_t n,
                        double* probs, uint8_t* actions) {
    return gbxcu_forward(c, params, feat, n, probs, actions, GBXCU_FWD_FAST);
}

int gbxcu_sample_batch(gbxcu_ctx* c, const float* params, const float* feat, size_t n,
                       uint64_t rng_state, uint8_t* actions) {
    if (!c || !params || (n && !feat) || !actions) return fail(GBXCU_EINVAL, "null argument");
    if (n == 0) return GBXCU_OK;
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    RET(upload(c->params, params, NP, st));
    RET(upload(c->feat, feat, n * F, st));
    RET(upload(c->seg_seed, &rng_state, 1, st));
    RET(c->actions.ensure(n));
    RET(run_forward(c, c->params.as<float>(), c->feat.as<float>(), n, nullptr,
                    c->actions.as<uint8_t>(), GBXCU_FWD_FAST, nullptr, 0,
                    c->seg_seed.as<uint64_t>(), 0.0, st, c->recheck, c->counters, c->flags,
                    FWD_SAMPLE));
    RET(check_flags(c->flags, st));
    CK(cudaMemcpyAsync(actions, c->actions.p, n, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return GBXCU_OK;
}

int gbxcu_collect_dev(gbxcu_ctx* c, const float* d_params, const float* d_feat,
                      const uint64_t* d_seg_off, size_t nseg, const uint64_t* d_seg_seed,
                      size_t n_states, double eps, uint8_t* d_actions, void* stream) {
    if (!c || !d_params || !d_seg_off || !d_seg_seed || !d_actions)
        return fail(GBXCU_EINVAL, "null argument");
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    return run_forward(c, d_params, d_feat, n_states, nullptr, d_actions, GBXCU_FWD_FAST, d_seg_off,
                       nseg, d_seg_seed, eps, pick(c, stream), c->recheck, c->counters, c->flags);
}

static int batch_grad(gbxcu_ctx* c, const float* params, const float* feat, const double* tgt,
                      size_t n, double* grad_out, double* loss_out) {
    if (!c || !params || !feat || !tgt) return fail(GBXCU_EINVAL, "null argument");
    if (n == 0) return fail(GBXCU_EINVAL, "empty batch");
    if (n > 0x7FFFFFFFull) return fail(GBXCU_EINVAL, "batch too large");
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    RET(upload(c->params, params, NP, st));
    RET(upload(c->feat, feat, n * F, st));
    RET(upload(c->tgt, tgt, n * 2, st));
    RET(c->order.ensure(n * 4));
    RET(c->grad.ensure(sizeof(double) * (NP + 1)));
    iota_kernel<<<std::max(1, std::min<int>((int)((n + 255) / 256), c->num_sms * 8)), 256, 0, st>>>(
        c->order.as<uint32_t>(), n);
    RET(check_launch(c, "iota_kernel"));
    TrainArgs a{};
    a.feat = c->feat.as<float>();
    a.tgt = c->tgt.as<double>();
    a.order = c->order.as<uint32_t>();
    a.params = c->params.as<float>();
    a.n = n;
    a.batch = (int)n;
    a.rank = 0;
    a.nranks = 1;
    double* dg = c->grad.as<double>();
    batch_grad_kernel<<<1, TRAIN_BLOCK, train_smem_bytes(64), st>>>(a, dg, dg + NP);
    RET(check_launch(c, "batch_grad_kernel"));
    if (grad_out) CK(cudaMemcpyAsync(grad_out, dg, sizeof(double) * NP, cudaMemcpyDeviceToHost, st));
    if (loss_out) CK(cudaMemcpyAsync(loss_out, dg + NP, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return GBXCU_OK;
}

int gbxcu_batch_kl_loss(gbxcu_ctx* c, const float* params, const float* feat, const double* tgt,
                        size_t n, double* loss_out) {
    return batch_grad(c, params, feat, tgt, n, nullptr, loss_out);
}

int gbxcu_batch_kl_gradient(gbxcu_ctx* c, const float* params, const float* feat,
                            const double* tgt, size_t n, double* grad_out) {
    return batch_grad(c, params, feat, tgt, n, grad_out, nullptr);
}

int gbxcu_fit(gbxcu_ctx* c, float* params_inout, const float* feat, const double* tgt, size_t n,
              const gbxcu_train_cfg* cfg, double* epoch_loss_out, int* diverged_epoch) {
    if (!c || !params_inout) return fail(GBXCU_EINVAL, "null argument");
    RET(validate_cfg(cfg, n));
    if (!feat || !tgt) return fail(GBXCU_EINVAL, "null dataset");
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    // the epoch-0 permutation needs no data: replay it on the side stream while
    // the log crosses PCIe, join before the first train launch
    RET(setup_kernel_attrs());
    RET(prepare_order(c, n, c->side));
    RET(shuffle_epoch(c, n, cfg->seed, 0, c->side));
    CK(cudaEventRecord(c->side_ev, c->side));
    RET(upload(c->params, params_inout, NP, st));
    RET(upload(c->feat, feat, n * F, st));
    RET(upload(c->tgt, tgt, n * 2, st));
    CK(cudaStreamWaitEvent(st, c->side_ev, 0));
    int rc = fit_device(c, c->params.as<float>(), c->feat.as<float>(), c->tgt.as<double>(), n, cfg,
                        epoch_loss_out, diverged_epoch, st, /*pre_shuffled=*/true);
    if (rc != GBXCU_OK && rc != GBXCU_EDIVERGED) return rc;
    const std::string msg = g_err;
    CK(cudaMemcpyAsync(params_inout, c->params.p, sizeof(float) * NP, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    g_err = msg;
    return rc;
}

int gbxcu_fit_dev(gbxcu_ctx* c, float* d_params, const float* d_feat, const double* d_tgt,
                  size_t n, const gbxcu_train_cfg* cfg, double* epoch_loss_out,
                  int* diverged_epoch, void* stream) {
    if (!c || !d_params || !d_feat || !d_tgt) return fail(GBXCU_EINVAL, "null argument");
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    return fit_device(c, d_params, d_feat, d_tgt, n, cfg, epoch_loss_out, diverged_epoch,
                      pick(c, stream));
}

int gbxcu_fit_order(gbxcu_ctx* c, size_t n, uint64_t seed, int epochs, uint32_t* order_out) {
    if (!c || !order_out) return fail(GBXCU_EINVAL, "null argument");
    if (n == 0) return GBXCU_OK;
    if (n > 0x7FFFFFFFull) return fail(GBXCU_EINVAL, "n too large");
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    RET(prepare_order(c, n, st));
    for (int e = 0; e < epochs; ++e) RET(shuffle_epoch(c, n, seed, e, st));
    CK(cudaMemcpyAsync(order_out, c->order.p, n * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return GBXCU_OK;
}

int gbxcu_comm_unique_id(uint8_t id_out[GBXCU_COMM_ID_BYTES]) {
    static_assert(sizeof(ncclUniqueId) == GBXCU_COMM_ID_BYTES, "ncclUniqueId size");
    ncclUniqueId id;
    CKN(ncclGetUniqueId(&id));
    std::memcpy(id_out, &id, sizeof(id));
    return GBXCU_OK;
}

int gbxcu_comm_init(gbxcu_ctx* c, const uint8_t id[GBXCU_COMM_ID_BYTES], int nranks, int rank) {
    if (!c || !id || nranks < 1 || rank < 0 || rank >= nranks)
        return fail(GBXCU_EINVAL, "bad communicator arguments");
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    if (c->comm) {
        ncclCommDestroy(c->comm);
        c->comm = nullptr;
    }
    // nranks == 1 still builds a (trivial) communicator: fit then runs the
    // data-parallel step sequence (partials -> reduce -> all-reduce -> update),
    // which is how that path is exercised on a single-GPU box.
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    CKN(ncclCommInitRank(&c->comm, nranks, uid, rank));
    c->nranks = nranks;
    c->rank = rank;
    return GBXCU_OK;
}

int gbxcu_peer_export(gbxcu_ctx* c, uint8_t handle_out[GBXCU_PEER_HANDLE_BYTES]) {
    static_assert(sizeof(cudaIpcMemHandle_t) == GBXCU_PEER_HANDLE_BYTES, "IPC handle size");
    if (!c || !handle_out) return fail(GBXCU_EINVAL, "null argument");
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    // sized for the largest grid (one CTA per SM); zeroed: counters start at 0
    if (c->xchg[0].cap < xchg_bytes(c->num_sms)) {
        if (c->xchg[0].p) CK(cudaFree(c->xchg[0].p));
        c->xchg[0].p = nullptr;
        c->xchg[0].cap = 0;
        RET(c->xchg[0].ensure(xchg_bytes(c->num_sms)));
    }
    CK(cudaMemset(c->xchg[0].p, 0, xchg_bytes(c->num_sms)));
    CK(cudaDeviceSynchronize());
    c->ctr_base[0] = 0;
    c->tag_next = 0;
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, c->xchg[0].p));
    std::memcpy(handle_out, &h, sizeof(h));
    return GBXCU_OK;
}

int gbxcu_peer_attach(gbxcu_ctx* c, int nranks, int rank, const uint8_t* handles) {
    if (!c || !handles || nranks < 2 || nranks > MAX_PEERS || rank < 0 || rank >= nranks)
        return fail(GBXCU_EINVAL, "bad peer-set arguments (2..8 ranks)");
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    if (c->comm) return fail(GBXCU_EINVAL, "detach the NCCL communicator first");
    if (c->xchg[0].cap < xchg_bytes(c->num_sms)) return fail(GBXCU_EINVAL, "call gbxcu_peer_export first");
    for (int r = 0; r < nranks; ++r) {
        if (r == rank) continue;
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handles + (size_t)r * GBXCU_PEER_HANDLE_BYTES, sizeof(h));
        CK(cudaIpcOpenMemHandle(&c->peer_ptr[r], h, cudaIpcMemLazyEnablePeerAccess));
    }
    c->peers = nranks;
    c->prank = rank;
    c->nranks = nranks;
    c->rank = rank;
    return GBXCU_OK;
}

int gbxcu_peer_detach(gbxcu_ctx* c) {
    if (!c) return fail(GBXCU_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    for (int r = 0; r < MAX_PEERS; ++r) {
        if (c->peer_ptr[r]) cudaIpcCloseMemHandle(c->peer_ptr[r]);
        c->peer_ptr[r] = nullptr;
    }
    c->peers = 1;
    c->prank = 0;
    c->nranks = 1;
    c->rank = 0;
    return GBXCU_OK;
}

int gbxcu_comm_destroy(gbxcu_ctx* c) {
    if (!c) return fail(GBXCU_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(c->mu);
    if (c->comm) CKN(ncclCommDestroy(c->comm));
    c->comm = nullptr;
    c->nranks = 1;
    c->rank = 0;
    return GBXCU_OK;
}

// ================================================================= Q-table
int gbxcu_qtable_create(gbxcu_ctx* c, double alpha, double omega, gbxcu_qtable** out) {
    if (!c || !out) return fail(GBXCU_EINVAL, "null argument");
    // QHyperparams::validate (proj/src/qtable.cpp:57-64)
    if (!(alpha > 0.0 && alpha <= 1.0)) return fail(GBXCU_EINVAL, "alpha must be in (0, 1]");
    if (!(omega > 0.0 && omega <= 1.0)) return fail(GBXCU_EINVAL, "omega must be in (0, 1]");
    auto* t = new gbxcu_qtable;
    t->ctx = c;
    t->alpha = alpha;
    t->omega = omega;
    // every store operation runs on the context stream: its buffers grow
    // through the stream-ordered pool (the table grows a little per call)
    for (DevBuf* b : {&t->keys, &t->q, &t->t, &t->cnt, &t->has, &t->nkeys, &t->nq, &t->nt,
                      &t->ncnt, &t->nhas, &t->bkeys, &t->bact, &t->brew, &t->bnow, &t->init_ids,
                      &t->count, &t->perm, &t->perm2, &t->digit, &t->digit2, &t->seg_head,
                      &t->key_head, &t->seg_scan, &t->key_scan, &t->seg_start, &t->seg_key,
                      &t->spread, &t->bad, &t->temp, &t->flag, &t->row, &t->rowkey, &t->sfeat,
                      &t->stgt, &t->bad_stage, &t->enc_tab, &t->rn})
        b->astream = c->stream;
    *out = t;
    return GBXCU_OK;
}

void gbxcu_qtable_free(gbxcu_qtable* t) { delete t; }

int gbxcu_qtable_clear(gbxcu_qtable* t) {
    if (!t) return fail(GBXCU_EINVAL, "null table");
    std::lock_guard<std::mutex> lk(t->ctx->mu);
    t->m = 0;  // device buffers are kept for the next fold
    return GBXCU_OK;
}

int gbxcu_qtable_size(const gbxcu_qtable* t, size_t* states, size_t* entries) {
    if (!t) return fail(GBXCU_EINVAL, "null table");
    std::lock_guard<std::mutex> lk(t->ctx->mu);
    CK(cudaSetDevice(t->ctx->device));
    if (states) *states = t->m;
    if (entries) {
        std::vector<uint8_t> h(2 * t->m);
        if (t->m) CK(cudaMemcpy(h.data(), t->has.p, 2 * t->m, cudaMemcpyDeviceToHost));
        size_t e = 0;
        for (uint8_t x : h) e += x;
        *entries = e;
    }
    return GBXCU_OK;
}

namespace {
int qtable_fold(gbxcu_qtable* t, const uint32_t* d_keys, const uint8_t* d_act, const double* d_rew,
                const uint64_t* d_now, size_t n, cudaStream_t st, size_t* bad_index) {
    gbxcu_ctx* c = t->ctx;
    // existing entries become init records
    size_t n_init = 0;
    RET(t->count.ensure(16));
    if (t->m) {
        RET(t->init_ids.ensure(sizeof(uint32_t) * 2 * t->m));
        CK(cudaMemsetAsync(t->count.p, 0, 8, st));
        qt_init_ids_kernel<<<c->num_sms * 4, 256, 0, st>>>(t->has.as<uint8_t>(), t->m,
                                                           t->init_ids.as<uint32_t>(),
                                                           t->count.as<unsigned long long>());
        RET(check_launch(c, "qt_init_ids_kernel"));
        unsigned long long k = 0;
        CK(cudaMemcpyAsync(&k, t->count.p, 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        n_init = (size_t)k;
        // entry ids in order (the atomics scatter them): sort is not needed for
        // correctness — the records' sort below orders them by key anyway
    }
    const size_t nrec = n_init + n;
    if (nrec == 0) return GBXCU_OK;
    if (nrec > 0xFFFFFFFFull) return fail(GBXCU_EINVAL, "q-table fold too large (> 2^32 records)");
    for (DevBuf* b : {&t->perm, &t->perm2, &t->seg_head, &t->key_head, &t->seg_scan, &t->key_scan,
                      &t->seg_start, &t->seg_key})
        RET(b->ensure(sizeof(uint32_t) * nrec));
    RET(t->digit.ensure(sizeof(unsigned long long) * nrec));   // packed 64-bit radix digits
    RET(t->digit2.ensure(sizeof(unsigned long long) * nrec));
    RET(t->spread.ensure(sizeof(uint32_t) * 64));
    RET(t->rn.ensure(16 * std::max<size_t>(n, 1)));
    RET(t->bad.ensure(16));
    const size_t tb = qt_temp_bytes(nrec);
    RET(t->temp.ensure(tb));
    QtFoldIO io{};
    io.tkeys = t->keys.as<uint32_t>();
    io.init = t->init_ids.as<uint32_t>();
    io.n_init = n_init;
    io.bkeys = d_keys;
    io.bact = d_act;
    io.reward = d_rew;
    io.now = d_now;
    io.n = n;
    io.limit = n;
    io.old_q = t->q.as<double>();
    io.old_t = t->t.as<uint64_t>();
    io.old_cnt = t->cnt.as<uint64_t>();
    io.alpha = t->alpha;
    io.omega = t->omega;
    io.perm = t->perm.as<uint32_t>();
    io.perm2 = t->perm2.as<uint32_t>();
    io.digit = t->digit.as<uint32_t>();
    io.digit2 = t->digit2.as<uint32_t>();
    io.seg_head = t->seg_head.as<uint32_t>();
    io.key_head = t->key_head.as<uint32_t>();
    io.seg_scan = t->seg_scan.as<uint32_t>();
    io.key_scan = t->key_scan.as<uint32_t>();
    io.seg_start = t->seg_start.as<uint32_t>();
    io.seg_key = t->seg_key.as<uint32_t>();
    io.spread = t->spread.as<uint32_t>();
    io.rn = t->rn.p;
    io.temp = t->temp.p;
    io.temp_bytes = tb;
    io.bad = t->bad.as<unsigned long long>();
    size_t nseg = 0, nkeys = 0;
    CK(qt_sort_segment(io, nseg, nkeys, c->num_sms, st));
    c->launches += 4;
    RET(t->nkeys.ensure(sizeof(uint32_t) * QT_KEY_WORDS * nkeys));
    RET(t->nq.ensure(sizeof(double) * 2 * nkeys));
    RET(t->nt.ensure(sizeof(uint64_t) * 2 * nkeys));
    RET(t->ncnt.ensure(sizeof(uint64_t) * 2 * nkeys));
    RET(t->nhas.ensure(2 * nkeys));
    CK(cudaMemsetAsync(t->nhas.p, 0, 2 * nkeys, st));
    CK(cudaMemsetAsync(t->bad.p, 0xFF, 8, st));
    CK(qt_fold(io, nseg, nkeys, t->nkeys.as<uint32_t>(), t->nq.as<double>(), t->nt.as<uint64_t>(),
               t->ncnt.as<uint64_t>(), t->nhas.as<uint8_t>(), c->num_sms, st));
    RET(check_launch(c, "qt_fold_kernel"));
    unsigned long long bad = ~0ull;
    CK(cudaMemcpyAsync(&bad, t->bad.p, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    *bad_index = bad == ~0ull ? (size_t)-1 : (size_t)bad;
    if (bad != ~0ull) return GBXCU_OK;  // caller re-folds the prefix
    for (auto pr : {std::make_pair(&t->keys, &t->nkeys), std::make_pair(&t->q, &t->nq),
                    std::make_pair(&t->t, &t->nt), std::make_pair(&t->cnt, &t->ncnt),
                    std::make_pair(&t->has, &t->nhas)}) {
        std::swap(pr.first->p, pr.second->p);  // DevBuf owns p: swap members, not objects
        std::swap(pr.first->cap, pr.second->cap);
    }
    t->m = nkeys;
    return GBXCU_OK;
}

int qtable_update(gbxcu_qtable* t, const uint32_t* d_keys, const uint8_t* d_act, const double* d_rew,
                  const uint64_t* d_now, size_t n, cudaStream_t st, size_t* bad_index) {
    size_t bad = (size_t)-1;
    RET(qtable_fold(t, d_keys, d_act, d_rew, d_now, n, st, &bad));
    if (bad == (size_t)-1) return GBXCU_OK;
    // ClockRegressionError at tuple `bad`: the reference has applied every
    // tuple before it (updates are sequential) — fold exactly that prefix.
    size_t bad2 = (size_t)-1;
    if (bad > 0) RET(qtable_fold(t, d_keys, d_act, d_rew, d_now, bad, st, &bad2));
    if (bad_index) *bad_index = bad;
    return fail(GBXCU_ECLOCK, "q_update check-in precedes the entry timestamp (tuple " +
                                  std::to_string(bad) + ")");
}
}  // namespace

int gbxcu_qtable_update_batch(gbxcu_qtable* t, const uint32_t* keys, const uint8_t* actions,
                              const double* rewards, const uint64_t* now, size_t n,
                              size_t* bad_index) {
    if (!t || (n && (!keys || !actions || !rewards || !now))) return fail(GBXCU_EINVAL, "null argument");
    if (bad_index) *bad_index = (size_t)-1;
    for (size_t i = 0; i < n; ++i)
        if (actions[i] > 1) return fail(GBXCU_EINVAL, "action must be 0 (wave32) or 1 (wave64)");
    if (n == 0) return GBXCU_OK;
    gbxcu_ctx* c = t->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    RET(upload(t->bkeys, keys, n * QT_KEY_WORDS, st));
    RET(upload(t->bact, actions, n, st));
    RET(upload(t->brew, rewards, n, st));
    RET(upload(t->bnow, now, n, st));
    return qtable_update(t, t->bkeys.as<uint32_t>(), t->bact.as<uint8_t>(), t->brew.as<double>(),
                         t->bnow.as<uint64_t>(), n, st, bad_index);
}

int gbxcu_qtable_update_batch_dev(gbxcu_qtable* t, const uint32_t* d_keys, const uint8_t* d_actions,
                                  const double* d_rewards, const uint64_t* d_now, size_t n,
                                  size_t* bad_index) {
    if (!t || (n && (!d_keys || !d_actions || !d_rewards || !d_now)))
        return fail(GBXCU_EINVAL, "null argument");
    if (bad_index) *bad_index = (size_t)-1;
    if (n == 0) return GBXCU_OK;
    gbxcu_ctx* c = t->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    return qtable_update(t, d_keys, d_actions, d_rewards, d_now, n, c->stream, bad_index);
}

int gbxcu_qtable_import(gbxcu_qtable* t, const uint32_t* keys, const double* q, const uint64_t* ts,
                        const uint64_t* cnt, const uint8_t* has, size_t m) {
    if (!t || (m && (!keys || !q || !ts || !cnt || !has))) return fail(GBXCU_EINVAL, "null argument");
    // the device table is a sorted set: keys strictly increasing (lexicographic)
    for (size_t r = 1; r < m; ++r) {
        const uint32_t* a = keys + (r - 1) * QT_KEY_WORDS;
        const uint32_t* b = keys + r * QT_KEY_WORDS;
        if (!std::lexicographical_compare(a, a + QT_KEY_WORDS, b, b + QT_KEY_WORDS))
            return fail(GBXCU_EINVAL, "imported keys must be strictly increasing");
    }
    gbxcu_ctx* c = t->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    RET(upload(t->keys, keys, m * QT_KEY_WORDS, st));
    RET(upload(t->q, q, 2 * m, st));
    RET(upload(t->t, ts, 2 * m, st));
    RET(upload(t->cnt, cnt, 2 * m, st));
    RET(upload(t->has, has, 2 * m, st));
    CK(cudaStreamSynchronize(st));
    t->m = m;
    return GBXCU_OK;
}

int gbxcu_qtable_export(const gbxcu_qtable* t, uint32_t* keys, double* q, uint64_t* ts, uint64_t* cnt,
                        uint8_t* has) {
    if (!t) return fail(GBXCU_EINVAL, "null table");
    std::lock_guard<std::mutex> lk(t->ctx->mu);
    CK(cudaSetDevice(t->ctx->device));
    const size_t m = t->m;
    if (!m) return GBXCU_OK;
    if (keys) CK(cudaMemcpy(keys, t->keys.p, sizeof(uint32_t) * QT_KEY_WORDS * m, cudaMemcpyDeviceToHost));
    if (q) CK(cudaMemcpy(q, t->q.p, sizeof(double) * 2 * m, cudaMemcpyDeviceToHost));
    if (ts) CK(cudaMemcpy(ts, t->t.p, sizeof(uint64_t) * 2 * m, cudaMemcpyDeviceToHost));
    if (cnt) CK(cudaMemcpy(cnt, t->cnt.p, sizeof(uint64_t) * 2 * m, cudaMemcpyDeviceToHost));
    if (has) CK(cudaMemcpy(has, t->has.p, 2 * m, cudaMemcpyDeviceToHost));
    return GBXCU_OK;
}

// ------------------------------------------------ columnar table file (f2)
namespace {
constexpr char QT_MAGIC[8] = {'G', 'B', 'X', 'Q', 'T', 'A', 'B', '\0'};
struct QtFileHeader {  // 64 bytes, little-endian
    char magic[8];
    uint32_t version, key_words;
    uint64_t m;
    double alpha, omega;
    uint64_t payload_bytes, checksum;
    uint64_t reserved;
};
static_assert(sizeof(QtFileHeader) == 64, "header layout");
size_t qt_align64(size_t b) { return (b + 63) & ~(size_t)63; }
// FNV-1a over 64-bit little-endian words (the tail zero-padded)
uint64_t qt_checksum(const unsigned char* p, size_t n) {
    uint64_t h = 0xcbf29ce484222325ull;
    size_t i = 0;
    for (; i + 8 <= n; i += 8) {
        uint64_t w;
        std::memcpy(&w, p + i, 8);
        h = (h ^ w) * 0x100000001b3ull;
    }
    if (i < n) {
        uint64_t w = 0;
        std::memcpy(&w, p + i, n - i);
        h = (h ^ w) * 0x100000001b3ull;
    }
    return h;
}
struct QtSections {
    size_t keys, q, t, cnt, has, total;
};
QtSections qt_sections(size_t m) {
    QtSections s{};
    s.keys = 0;
    s.q = qt_align64(s.keys + sizeof(uint32_t) * QT_KEY_WORDS * m);
    s.t = qt_align64(s.q + sizeof(double) * 2 * m);
    s.cnt = qt_align64(s.t + sizeof(uint64_t) * 2 * m);
    s.has = qt_align64(s.cnt + sizeof(uint64_t) * 2 * m);
    s.total = qt_align64(s.has + 2 * m);
    return s;
}
}  // namespace

int gbxcu_qtable_save_columnar(const gbxcu_qtable* t, const char* path) {
    if (!t || !path) return fail(GBXCU_EINVAL, "null argument");
    const size_t m = t->m;
    const QtSections sec = qt_sections(m);
    std::vector<unsigned char> buf;
    try {
        buf.assign(sizeof(QtFileHeader) + sec.total, 0);
    } catch (const std::bad_alloc&) {
        return fail(GBXCU_EINVAL, "q-table too large for host memory");
    }
    unsigned char* pay = buf.data() + sizeof(QtFileHeader);
    RET(gbxcu_qtable_export(t, reinterpret_cast<uint32_t*>(pay + sec.keys),
                            reinterpret_cast<double*>(pay + sec.q), reinterpret_cast<uint64_t*>(pay + sec.t),
                            reinterpret_cast<uint64_t*>(pay + sec.cnt), pay + sec.has));
    {  // absent entries carry no state: zero them so files are deterministic
        uint8_t* has = pay + sec.has;
        double* q = reinterpret_cast<double*>(pay + sec.q);
        uint64_t* ts = reinterpret_cast<uint64_t*>(pay + sec.t);
        uint64_t* cn = reinterpret_cast<uint64_t*>(pay + sec.cnt);
        for (size_t e = 0; e < 2 * m; ++e)
            if (!has[e]) q[e] = 0.0, ts[e] = 0, cn[e] = 0;
    }
    QtFileHeader h{};
    std::memcpy(h.magic, QT_MAGIC, 8);
    h.version = 1;
    h.key_words = QT_KEY_WORDS;
    h.m = m;
    h.alpha = t->alpha;
    h.omega = t->omega;
    h.payload_bytes = sec.total;
    h.checksum = qt_checksum(pay, sec.total);
    std::memcpy(buf.data(), &h, sizeof(h));
    FILE* f = std::fopen(path, "wb");
    if (!f) return fail(GBXCU_EINVAL, std::string("cannot open for writing: ") + path);
    const bool ok = std::fwrite(buf.data(), 1, buf.size(), f) == buf.size();
    if (std::fclose(f) != 0 || !ok) return fail(GBXCU_EINVAL, std::string("write failed: ") + path);
    return GBXCU_OK;
}

int gbxcu_qtable_load_columnar(gbxcu_qtable* t, const char* path) {
    if (!t || !path) return fail(GBXCU_EINVAL, "null argument");
    FILE* f = std::fopen(path, "rb");
    if (!f) return fail(GBXCU_EINVAL, std::string("cannot open: ") + path);
    QtFileHeader h{};
    const bool got = std::fread(&h, 1, sizeof(h), f) == sizeof(h);
    if (!got || std::memcmp(h.magic, QT_MAGIC, 8) != 0) {
        std::fclose(f);
        return fail(GBXCU_EINVAL, "not a columnar q-table file");
    }
    if (h.version != 1 || h.key_words != QT_KEY_WORDS) {
        std::fclose(f);
        return fail(GBXCU_EINVAL, "unsupported columnar q-table format version");
    }
    // QHyperparams::validate (proj/src/qtable.cpp:57-64), as QTable::load does
    if (!(h.alpha > 0.0 && h.alpha <= 1.0) || !(h.omega > 0.0 && h.omega <= 1.0)) {
        std::fclose(f);
        return fail(GBXCU_EINVAL, "columnar q-table holds invalid hyperparameters");
    }
    if (h.m > (size_t)1 << 32) {
        std::fclose(f);
        return fail(GBXCU_EINVAL, "columnar q-table too large");
    }
    const QtSections sec = qt_sections((size_t)h.m);
    if (h.payload_bytes != sec.total) {
        std::fclose(f);
        return fail(GBXCU_EINVAL, "columnar q-table size does not match its header");
    }
    // the file must hold exactly header + payload before anything is allocated
    // (a corrupt m must not turn into a huge allocation)
    if (std::fseek(f, 0, SEEK_END) != 0) {
        std::fclose(f);
        return fail(GBXCU_EINVAL, "cannot seek in columnar q-table file");
    }
    const long fsize = std::ftell(f);
    if (fsize < 0 || (unsigned long)fsize != sizeof(QtFileHeader) + sec.total ||
        std::fseek(f, (long)sizeof(QtFileHeader), SEEK_SET) != 0) {
        std::fclose(f);
        return fail(GBXCU_EINVAL, "columnar q-table truncated or has trailing bytes");
    }
    std::vector<unsigned char> pay;
    try {
        pay.resize(sec.total);
    } catch (const std::bad_alloc&) {
        std::fclose(f);
        return fail(GBXCU_EINVAL, "columnar q-table too large for host memory");
    }
    const bool full = std::fread(pay.data(), 1, sec.total, f) == sec.total;
    const bool at_end = std::fgetc(f) == EOF;
    std::fclose(f);
    if (!full || !at_end) return fail(GBXCU_EINVAL, "columnar q-table truncated or has trailing bytes");
    if (qt_checksum(pay.data(), sec.total) != h.checksum)
        return fail(GBXCU_EINVAL, "columnar q-table checksum mismatch");
    const uint8_t* has = pay.data() + sec.has;
    const uint64_t* cnt = reinterpret_cast<const uint64_t*>(pay.data() + sec.cnt);
    for (size_t e = 0; e < 2 * (size_t)h.m; ++e) {
        if (has[e] > 1) return fail(GBXCU_EINVAL, "columnar q-table: bad presence flag");
        if (has[e] && cnt[e] == 0) return fail(GBXCU_EINVAL, "columnar q-table: entry with zero updates");
    }
    RET(gbxcu_qtable_import(t, reinterpret_cast<const uint32_t*>(pay.data() + sec.keys),
                            reinterpret_cast<const double*>(pay.data() + sec.q),
                            reinterpret_cast<const uint64_t*>(pay.data() + sec.t), cnt, has, (size_t)h.m));
    t->alpha = h.alpha;
    t->omega = h.omega;
    return GBXCU_OK;
}

namespace {
int qtable_snapshot(gbxcu_qtable* t, double rho, float* d_feat, double* d_tgt, size_t cap, size_t* rows,
                    cudaStream_t st) {
    gbxcu_ctx* c = t->ctx;
    if (!(rho > 0.0)) return fail(GBXCU_ETEMPERATURE, "softmax temperature must be positive");
    *rows = 0;
    const size_t m = t->m;
    if (m == 0) return GBXCU_OK;
    RET(t->flag.ensure(sizeof(uint32_t) * m));
    RET(t->row.ensure(sizeof(uint32_t) * m));
    RET(t->bad_stage.ensure(16));
    const size_t tb = qt_temp_bytes(m);
    RET(t->temp.ensure(tb));
    qt_both_kernel<<<c->num_sms * 4, 256, 0, st>>>(t->has.as<uint8_t>(), m, t->flag.as<uint32_t>());
    RET(check_launch(c, "qt_both_kernel"));
    CK(qt_exclusive_scan(t->temp.p, tb, t->flag.as<uint32_t>(), t->row.as<uint32_t>(), m, st));
    uint32_t tail[2];
    CK(cudaMemcpyAsync(&tail[0], t->row.as<uint32_t>() + m - 1, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&tail[1], t->flag.as<uint32_t>() + m - 1, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const size_t r = (size_t)tail[0] + tail[1];
    *rows = r;
    if (!d_feat) return GBXCU_OK;  // size query
    if (r > cap) return fail(GBXCU_EINVAL, "snapshot buffers too small");
    CK(cudaMemsetAsync(t->bad_stage.p, 0, 4, st));
    if (r == 0) return GBXCU_OK;
    RET(t->rowkey.ensure(sizeof(uint32_t) * r));
    qt_rowkey_kernel<<<c->num_sms * 4, 256, 0, st>>>(t->flag.as<uint32_t>(), t->row.as<uint32_t>(), m,
                                                     t->rowkey.as<uint32_t>());
    RET(check_launch(c, "qt_rowkey_kernel"));
    if (!t->enc_ready) {
        RET(t->enc_tab.ensure(sizeof(float) * QT_ENC_TAB));
        qt_enc_table_kernel<<<QT_ENC_TAB / 256, 256, 0, st>>>(t->enc_tab.as<float>());
        RET(check_launch(c, "qt_enc_table_kernel"));
        t->enc_ready = true;
    }
    const int sgrid = (int)std::min<size_t>((r + 127) / 128, (size_t)c->num_sms * 5);  // 5 CTAs/SM (smem)
    qt_snapshot_kernel<<<sgrid, 128, 0, st>>>(t->keys.as<uint32_t>(), t->q.as<double>(),
                                              t->rowkey.as<uint32_t>(), r, rho, t->enc_tab.as<float>(),
                                              d_feat, d_tgt, t->bad_stage.as<int>());
    RET(check_launch(c, "qt_snapshot_kernel"));
    int bs = 0;
    CK(cudaMemcpyAsync(&bs, t->bad_stage.p, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (bs) return fail(GBXCU_EINVAL, "state key holds invalid stage index");
    return GBXCU_OK;
}
}  // namespace

int gbxcu_qtable_snapshot(gbxcu_qtable* t, double rho, float* feat, double* tgt, size_t cap, size_t* rows) {
    if (!t || !rows) return fail(GBXCU_EINVAL, "null argument");
    gbxcu_ctx* c = t->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    size_t r = 0;
    RET(qtable_snapshot(t, rho, nullptr, nullptr, 0, &r, st));
    *rows = r;
    if (!feat) return GBXCU_OK;
    if (r > cap) return fail(GBXCU_EINVAL, "snapshot buffers too small");
    RET(t->sfeat.ensure(sizeof(float) * F * std::max<size_t>(r, 1)));
    RET(t->stgt.ensure(sizeof(double) * 2 * std::max<size_t>(r, 1)));
    RET(qtable_snapshot(t, rho, t->sfeat.as<float>(), t->stgt.as<double>(), r, &r, st));
    CK(cudaMemcpyAsync(feat, t->sfeat.p, sizeof(float) * F * r, cudaMemcpyDeviceToHost, st));
    if (tgt) CK(cudaMemcpyAsync(tgt, t->stgt.p, sizeof(double) * 2 * r, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return GBXCU_OK;
}

int gbxcu_qtable_snapshot_dev(gbxcu_qtable* t, double rho, float* d_feat, double* d_tgt, size_t cap,
                              size_t* rows) {
    if (!t || !rows) return fail(GBXCU_EINVAL, "null argument");
    gbxcu_ctx* c = t->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    return qtable_snapshot(t, rho, d_feat, d_tgt, cap, rows, c->stream);
}

int gbxcu_aggregate(gbxcu_ctx* c, const gbxcu_suite* s, const uint8_t* shader_actions,
                    const uint64_t* run_seed, int n_samples, double* rows_out,
                    double* samples_out) {
    if (!c || !shader_actions || !run_seed || !rows_out) return fail(GBXCU_EINVAL, "null argument");
    RET(suite_args(s));
    if (n_samples < 1) return fail(GBXCU_EINVAL, "sample count must be >= 1");
    if (s->n_apps == 0) return GBXCU_OK;
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    RET(upload(c->s_app_pipe, s->app_pipe_off, s->n_apps + 1, st));
    RET(upload(c->s_pipe_slot, s->pipe_slot_off, s->n_pipes + 1, st));
    RET(upload(c->s_slot_shader, s->slot_shader, s->n_slots, st));
    RET(upload(c->s_slot_frac, s->slot_frac, s->n_slots, st));
    RET(upload(c->s_pipe_wt, s->pipe_wt, s->n_pipes * 2, st));
    RET(upload(c->s_shader_lat, s->shader_lat, s->n_shaders * 3, st));
    RET(upload(c->s_app_f64, s->app_f64, s->n_apps * 4, st));
    RET(upload(c->s_actions, shader_actions, s->n_shaders, st));
    RET(upload(c->s_run_seed, run_seed, s->n_apps, st));
    RET(c->s_rows.ensure(sizeof(double) * 5 * s->n_apps));
    RET(c->s_samples.ensure(samples_out ? sizeof(double) * s->n_apps * n_samples : 16));
    AggArgs a{};
    a.n_apps = s->n_apps;
    a.app_pipe_off = c->s_app_pipe.as<uint64_t>();
    a.pipe_slot_off = c->s_pipe_slot.as<uint64_t>();
    a.slot_shader = c->s_slot_shader.as<uint32_t>();
    a.slot_frac = c->s_slot_frac.as<double>();
    a.pipe_wt = c->s_pipe_wt.as<double>();
    a.shader_lat = c->s_shader_lat.as<double>();
    a.app_f64 = c->s_app_f64.as<double>();
    a.shader_action = c->s_actions.as<uint8_t>();
    a.run_seed = c->s_run_seed.as<uint64_t>();
    a.n_samples = n_samples;
    a.rows = c->s_rows.as<double>();
    a.samples = samples_out ? c->s_samples.as<double>() : nullptr;
    RET(launch_aggregate(c, a, st));
    CK(cudaMemcpyAsync(rows_out, c->s_rows.p, sizeof(double) * 5 * s->n_apps,
                       cudaMemcpyDeviceToHost, st));
    if (samples_out)
        CK(cudaMemcpyAsync(samples_out, c->s_samples.p, sizeof(double) * s->n_apps * n_samples,
                           cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return GBXCU_OK;
}

static int run_histogram(gbxcu_ctx* c, const double* d_rows, int stride, size_t n, DevBuf& lower,
                         DevBuf& count, DevBuf& nbins, size_t cap, double* lower_out,
                         uint64_t* count_out, size_t* n_bins, cudaStream_t st) {
    RET(lower.ensure(sizeof(double) * std::max<size_t>(cap, 1)));
    RET(count.ensure(sizeof(uint64_t) * std::max<size_t>(cap, 1)));
    RET(nbins.ensure(16));
    histogram_kernel<<<1, 1024, 0, st>>>(d_rows, stride, n, lower.as<double>(),
                                         count.as<unsigned long long>(), cap,
                                         nbins.as<unsigned long long>());
    RET(check_launch(c, "histogram_kernel"));
    unsigned long long nb = 0;
    CK(cudaMemcpyAsync(&nb, nbins.p, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const size_t w = std::min<size_t>(nb, cap);
    if (w) {
        if (lower_out) CK(cudaMemcpyAsync(lower_out, lower.p, sizeof(double) * w, cudaMemcpyDeviceToHost, st));
        if (count_out) CK(cudaMemcpyAsync(count_out, count.p, sizeof(uint64_t) * w, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    }
    if (n_bins) *n_bins = nb;
    return GBXCU_OK;
}

int gbxcu_histogram(gbxcu_ctx* c, const double* uplift, size_t n, double* lower_out,
                    uint64_t* count_out, size_t cap, size_t* n_bins) {
    if (!c || (n && !uplift)) return fail(GBXCU_EINVAL, "null argument");
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    if (n == 0) {
        if (n_bins) *n_bins = 0;
        return GBXCU_OK;
    }
    // lay the uplifts out as rows of stride 5 (column 3), as the fused sweep does
    std::vector<double> rows(5 * n, 0.0);
    for (size_t k = 0; k < n; ++k) rows[5 * k + 3] = uplift[k];
    RET(upload(c->s_rows, rows.data(), rows.size(), st));
    return run_histogram(c, c->s_rows.as<double>(), 5, n, c->h_lower, c->h_count, c->h_nbins, cap,
                         lower_out, count_out, n_bins, st);
}

int gbxcu_suite_upload(gbxcu_ctx* c, const gbxcu_suite* s, const float* features,
                       gbxcu_dsuite** out) {
    if (!c || !out || !features) return fail(GBXCU_EINVAL, "null argument");
    RET(suite_args(s));
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    auto* d = new gbxcu_dsuite;
    d->ctx = c;
    d->n_apps = s->n_apps;
    d->n_pipes = s->n_pipes;
    d->n_slots = s->n_slots;
    d->n_shaders = s->n_shaders;
    int rc = GBXCU_OK;
    auto up = [&](int r) { if (rc == GBXCU_OK) rc = r; };
    up(upload(d->app_pipe, s->app_pipe_off, s->n_apps + 1, st));
    up(upload(d->pipe_slot, s->pipe_slot_off, s->n_pipes + 1, st));
    up(upload(d->slot_shader, s->slot_shader, s->n_slots, st));
    up(upload(d->slot_frac, s->slot_frac, s->n_slots, st));
    up(upload(d->pipe_wt, s->pipe_wt, s->n_pipes * 2, st));
    up(upload(d->shader_lat, s->shader_lat, s->n_shaders * 3, st));
    up(upload(d->app_f64, s->app_f64, s->n_apps * 4, st));
    up(upload(d->features, features, s->n_shaders * F, st));
    up(d->actions.ensure(std::max<size_t>(s->n_shaders, 1)));
    up(d->rows.ensure(sizeof(double) * 5 * std::max<size_t>(s->n_apps, 1)));
    if (rc == GBXCU_OK && cudaStreamSynchronize(st) != cudaSuccess)
        rc = fail(GBXCU_ECUDA, "suite upload failed");
    if (rc != GBXCU_OK) {
        delete d;
        return rc;
    }
    *out = d;
    return GBXCU_OK;
}

void gbxcu_suite_free(gbxcu_dsuite* s) { delete s; }

const float* gbxcu_suite_features(const gbxcu_dsuite* s) {
    return s ? s->features.as<float>() : nullptr;
}

static int evaluate_dev(gbxcu_ctx* c, const gbxcu_dsuite* s, const float* d_params,
                        int n_samples, uint64_t seed, uint8_t* d_actions, double* d_rows,
                        cudaStream_t st, DevBuf& recheck, DevBuf& counters, DevBuf& flags) {
    if (n_samples < 1) return fail(GBXCU_EINVAL, "sample count must be >= 1");
    CK(cudaEventRecord(c->eval_ev[0], st));
    RET(run_forward(c, d_params, s->features.as<float>(), s->n_shaders, nullptr, d_actions,
                    GBXCU_FWD_FAST, nullptr, 0, nullptr, 0.0, st, recheck, counters, flags));
    CK(cudaEventRecord(c->eval_ev[1], st));
    if (s->n_apps == 0) {
        CK(cudaEventRecord(c->eval_ev[2], st));
        return GBXCU_OK;
    }
    AggArgs a{};
    a.n_apps = s->n_apps;
    a.app_pipe_off = s->app_pipe.as<uint64_t>();
    a.pipe_slot_off = s->pipe_slot.as<uint64_t>();
    a.slot_shader = s->slot_shader.as<uint32_t>();
    a.slot_frac = s->slot_frac.as<double>();
    a.pipe_wt = s->pipe_wt.as<double>();
    a.shader_lat = s->shader_lat.as<double>();
    a.app_f64 = s->app_f64.as<double>();
    a.shader_action = d_actions;
    a.run_seed = nullptr;
    a.eval_seed = seed;
    a.n_samples = n_samples;
    a.rows = d_rows;
    a.samples = nullptr;
    RET(launch_aggregate(c, a, st));
    CK(cudaEventRecord(c->eval_ev[2], st));
    return GBXCU_OK;
}

// One app-range shard of evaluate (aggregation shards by app so
// no segment straddles GPUs): infers only the shaders the range's slots
// reference and aggregates apps [app_lo, app_hi) with their GLOBAL indices in
// the seeds, so gathering the shards' rows reproduces the unsharded rows bit
// for bit (the histogram is then built from the gathered uplifts).
int gbxcu_evaluate_shard(gbxcu_ctx* c, const gbxcu_dsuite* s, const float* params, int n_samples,
                         uint64_t seed, size_t app_lo, size_t app_hi, double* rows_out) {
    if (!c || !s || !params || (app_hi > app_lo && !rows_out)) return fail(GBXCU_EINVAL, "null argument");
    if (app_lo > app_hi || app_hi > s->n_apps) return fail(GBXCU_EINVAL, "app range out of bounds");
    if (n_samples < 1) return fail(GBXCU_EINVAL, "sample count must be >= 1");
    if (app_hi == app_lo) return GBXCU_OK;
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    gbxcu_dsuite* sm = const_cast<gbxcu_dsuite*>(s);
    RET(upload(sm->params, params, NP, st));
    RET(sm->actions.ensure(std::max<size_t>(1, s->n_shaders)));
    RET(sm->rows.ensure(sizeof(double) * 5 * (app_hi - app_lo)));
    // slot range of the apps, then the shader range those slots reference
    uint64_t pipes[2], slots[2];
    CK(cudaMemcpyAsync(&pipes[0], s->app_pipe.as<uint64_t>() + app_lo, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&pipes[1], s->app_pipe.as<uint64_t>() + app_hi, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    CK(cudaMemcpyAsync(&slots[0], s->pipe_slot.as<uint64_t>() + pipes[0], 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&slots[1], s->pipe_slot.as<uint64_t>() + pipes[1], 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    RET(sm->counters.ensure(16));
    unsigned int range[2] = {0xFFFFFFFFu, 0u};
    if (slots[1] > slots[0]) {
        CK(cudaMemcpyAsync(sm->counters.p, range, 8, cudaMemcpyHostToDevice, st));
        slot_shader_range_kernel<<<c->num_sms * 2, 256, 0, st>>>(s->slot_shader.as<uint32_t>(), slots[0],
                                                                 slots[1], sm->counters.as<unsigned int>());
        RET(check_launch(c, "slot_shader_range_kernel"));
        CK(cudaMemcpyAsync(range, sm->counters.p, 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (range[1] >= s->n_shaders) return fail(GBXCU_EINVAL, "slot references a missing shader");
        RET(run_forward(c, sm->params.as<float>(), s->features.as<float>() + (size_t)range[0] * F,
                        (size_t)range[1] - range[0] + 1, nullptr, sm->actions.as<uint8_t>() + range[0],
                        GBXCU_FWD_FAST, nullptr, 0, nullptr, 0.0, st, sm->recheck, sm->counters,
                        sm->flags));
        RET(check_flags(sm->flags, st));
    }
    AggArgs a{};
    a.n_apps = app_hi - app_lo;
    a.app_pipe_off = s->app_pipe.as<uint64_t>() + app_lo;
    a.pipe_slot_off = s->pipe_slot.as<uint64_t>();
    a.slot_shader = s->slot_shader.as<uint32_t>();
    a.slot_frac = s->slot_frac.as<double>();
    a.pipe_wt = s->pipe_wt.as<double>();
    a.shader_lat = s->shader_lat.as<double>();
    a.app_f64 = s->app_f64.as<double>() + 4 * app_lo;
    a.shader_action = sm->actions.as<uint8_t>();
    a.eval_seed = seed;
    a.n_samples = n_samples;
    a.rows = sm->rows.as<double>();
    a.app_base = app_lo;
    RET(launch_aggregate(c, a, st));
    CK(cudaMemcpyAsync(rows_out, sm->rows.p, sizeof(double) * 5 * a.n_apps, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return GBXCU_OK;
}

int gbxcu_evaluate(gbxcu_ctx* c, const gbxcu_dsuite* s, const float* params, int n_samples,
                   uint64_t seed, double* rows_out, uint8_t* shader_actions_out,
                   double* hist_lower, uint64_t* hist_count, size_t hist_cap, size_t* n_bins) {
    if (!c || !s || !params || !rows_out) return fail(GBXCU_EINVAL, "null argument");
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    gbxcu_dsuite* sm = const_cast<gbxcu_dsuite*>(s);
    RET(upload(sm->params, params, NP, st));
    RET(evaluate_dev(c, s, sm->params.as<float>(), n_samples, seed, sm->actions.as<uint8_t>(),
                     sm->rows.as<double>(), st, sm->recheck, sm->counters, sm->flags));
    RET(check_flags(sm->flags, st));
    if (s->n_apps)
        CK(cudaMemcpyAsync(rows_out, s->rows.p, sizeof(double) * 5 * s->n_apps,
                           cudaMemcpyDeviceToHost, st));
    if (shader_actions_out && s->n_shaders)
        CK(cudaMemcpyAsync(shader_actions_out, s->actions.p, s->n_shaders, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (hist_lower || hist_count || n_bins)
        RET(run_histogram(c, s->rows.as<double>(), 5, s->n_apps, sm->h_lower, sm->h_count,
                          sm->h_nbins, hist_cap, hist_lower, hist_count, n_bins, st));
    return GBXCU_OK;
}

int gbxcu_evaluate_dev(gbxcu_ctx* c, const gbxcu_dsuite* s, const float* d_params, int n_samples,
                       uint64_t seed, uint8_t* d_actions, double* d_rows, void* stream) {
    if (!c || !s || !d_params || !d_actions || !d_rows) return fail(GBXCU_EINVAL, "null argument");
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    gbxcu_dsuite* sm = const_cast<gbxcu_dsuite*>(s);
    return evaluate_dev(c, s, d_params, n_samples, seed, d_actions, d_rows, pick(c, stream),
                        sm->recheck, sm->counters, sm->flags);
}

}  // extern "C"

// =========================================================================
// Wide MLP (C4): 44 -> H -> H -> 2 on tcgen05 TF32 GEMMs (k_wide.cu).
namespace {

constexpr int kGemmTile = 128;  // GM == GN in k_wide.cu

size_t wide_param_count(int H) { return (size_t)H * F + H + (size_t)H * H + H + 2 * (size_t)H + 2; }

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                   CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                   CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}

// K-major fp32 operand [rows][ld] (K valid columns) as TMA boxes of
// {32 fp32 = 128 B, box_rows} with the 128-byte swizzle (tma_gemm_kernel).
bool make_operand_map(CUtensorMap* m, const float* base, int K, int rows, int ld, int box_rows) {
    const EncodeTiledFn enc = encode_tiled();
    if (!enc) return false;
    const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(float)};
    const cuuint32_t box[2] = {32, (cuuint32_t)box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN>
int launch_tma_gemm(gbxcu_ctx* c, const GemmArgs& g, int splits, cudaStream_t st, bool& done) {
    CUtensorMap ma, mb;
    done = make_operand_map(&ma, g.A, g.K, g.M, g.lda, TM_BM_HOST) &&
           make_operand_map(&mb, g.B, g.K, g.N, g.ldb, BN);
    if (!done) return GBXCU_OK;
    dim3 grid((g.N + BN - 1) / BN, (g.M + TM_BM_HOST - 1) / TM_BM_HOST, splits);
    tma_gemm_kernel<BN><<<grid, 128, tma_gemm_smem_bytes<BN>(), st>>>(ma, mb, g);
    return check_launch(c, "tma_gemm_kernel");
}

int launch_gemm(gbxcu_ctx* c, const GemmArgs& g, int splits, cudaStream_t st) {
    // TMA path: plain (non-gathered) operands with 16-byte row strides
    const bool tma_ok = !g.a_rows && g.K % 4 == 0 && g.lda % 4 == 0 && g.ldb % 4 == 0 &&
                        ((uintptr_t)g.A % 16) == 0 && ((uintptr_t)g.B % 16) == 0;
    if (tma_ok) {
        bool done = false;
        int rc;
        if (g.N <= 64) rc = launch_tma_gemm<64>(c, g, splits, st, done);
        else if (splits > 1 || g.N < 256) rc = launch_tma_gemm<128>(c, g, splits, st, done);
        else rc = launch_tma_gemm<256>(c, g, splits, st, done);
        if (rc != GBXCU_OK || done) return rc;
        // the wide path relies on TMA's zero fill past K (no tail clearing)
        return fail(GBXCU_ECUDA, "cuTensorMapEncodeTiled unavailable or rejected the operand");
    }
    dim3 grid((g.N + kGemmTile - 1) / kGemmTile, (g.M + kGemmTile - 1) / kGemmTile, splits);
    tc_gemm_kernel<<<grid, 128, gemm_smem_bytes(), st>>>(g);
    return check_launch(c, "tc_gemm_kernel");
}

int check_hidden(int H) {
    if (H < 32 || H > 1024 || H % 32 != 0)
        return fail(GBXCU_EINVAL, "wide MLP hidden width must be a multiple of 32 in [32, 1024]");
    return GBXCU_OK;
}

// Working set for batches of up to bmax rows per rank.
int wide_alloc(gbxcu_ctx* c, int H, size_t bmax, int splits4, int splits5, int rsplit) {
    const size_t ldt = (bmax + 3) & ~(size_t)3;
    RET(c->w_grad.ensure(sizeof(float) * wide_param_count(H)));
    RET(c->w_w1t.ensure(sizeof(float) * H * H));
    RET(c->w_h1.ensure(sizeof(float) * bmax * H));
    RET(c->w_h2.ensure(sizeof(float) * bmax * H));
    RET(c->w_d2.ensure(sizeof(float) * bmax * H));
    for (DevBuf* b : {&c->w_h1t, &c->w_d2t, &c->w_d1t}) RET(b->ensure(sizeof(float) * H * ldt));
    RET(c->w_xt.ensure(sizeof(float) * 48 * ldt));
    RET(c->w_xg.ensure(sizeof(float) * 48 * bmax));
    RET(c->w_w0p.ensure(sizeof(float) * 48 * H));
    RET(c->w_d3.ensure(sizeof(float) * 2 * bmax));
    RET(c->w_kl.ensure(sizeof(double) * bmax));
    RET(c->w_part.ensure(sizeof(double) * ((bmax + 31) / 32) * (3 * H + 3)));
    RET(c->w_g4.ensure(sizeof(float) * (size_t)splits4 * H * H));
    RET(c->w_g5.ensure(sizeof(float) * (size_t)splits5 * H * 48));
    RET(c->w_loss.ensure(64));
    return GBXCU_OK;
}

int blocks(size_t n, int t = 256) { return (int)std::max<size_t>(1, (n + t - 1) / t); }

// One SGD step on rows[0, nbr) (this rank's slice of a global batch of nb).
int wide_step(gbxcu_ctx* c, int H, float* P, const float* feat, const double* tgt,
              const uint32_t* rows, int nbr, size_t nb, size_t ldt, double lr, const int* epoch,
              int splits4, int splits5, int rsplit, cudaStream_t st) {
    const size_t o_b0 = (size_t)H * F, o_w1 = o_b0 + H, o_b1 = o_w1 + (size_t)H * H,
                 o_w2 = o_b1 + H;
    float* G = c->w_grad.as<float>();
    if (nbr > 0) {
        // (the K = batch GEMMs read exactly nbr columns through TMA, which
        //  zero-fills past the end: no tail clearing needed)
        wide_gather_xt_kernel<<<blocks(nbr), 256, 0, st>>>(feat, rows, nbr, c->w_xt.as<float>(), (int)ldt,
                                                           c->w_xg.as<float>());
        RET(check_launch(c, "wide_gather_xt_kernel"));

        GemmArgs g1{};  // H1 = relu(X W0^T + b0), also H1^T (X gathered, K padded to 48)
        g1.M = nbr; g1.N = H; g1.K = 48;
        g1.A = c->w_xg.as<float>(); g1.lda = 48;
        g1.B = c->w_w0p.as<float>(); g1.ldb = 48;
        g1.epi = EPI_BIAS_RELU; g1.bias = P + o_b0;
        g1.out = c->w_h1.as<float>(); g1.ldo = H;
        g1.out_t = c->w_h1t.as<float>(); g1.ldt = (int)ldt;
        RET(launch_gemm(c, g1, 1, st));

        GemmArgs g2{};  // H2 = relu(H1 W1^T + b1)
        g2.M = nbr; g2.N = H; g2.K = H;
        g2.A = c->w_h1.as<float>(); g2.lda = H;
        g2.B = P + o_w1; g2.ldb = H;
        g2.epi = EPI_BIAS_RELU; g2.bias = P + o_b1;
        g2.out = c->w_h2.as<float>(); g2.ldo = H;
        RET(launch_gemm(c, g2, 1, st));

        WideHeadArgs h{};
        h.h2 = c->w_h2.as<float>(); h.w2 = P + o_w2; h.b2 = P + o_w2 + 2 * H;
        h.tgt = tgt; h.rows = rows; h.nb = nbr; h.hidden = H; h.ldt = (int)ldt;
        h.inv_b = 1.0 / (double)nb;
        h.kl = c->w_kl.as<double>(); h.d3 = c->w_d3.as<float>();
        h.d2 = c->w_d2.as<float>(); h.d2t = c->w_d2t.as<float>();
        h.part = c->w_part.as<double>();
        wide_head_kernel<<<(nbr + 31) / 32, 1024, sizeof(float) * 32 * (H + 1), st>>>(h);
        RET(check_launch(c, "wide_head_kernel"));

        GemmArgs g3{};  // D1^T = ((D2 W1) . [H1 > 0])^T
        g3.M = nbr; g3.N = H; g3.K = H;
        g3.A = c->w_d2.as<float>(); g3.lda = H;
        g3.B = c->w_w1t.as<float>(); g3.ldb = H;
        g3.epi = EPI_MASK_T; g3.mask = c->w_h1.as<float>(); g3.ldm = H;
        g3.out_t = c->w_d1t.as<float>(); g3.ldt = (int)ldt;
        RET(launch_gemm(c, g3, 1, st));

        GemmArgs g4{};  // gW1 = D2^T H1 (split-K partials)
        g4.M = H; g4.N = H; g4.K = nbr;
        g4.A = c->w_d2t.as<float>(); g4.lda = (int)ldt;
        g4.B = c->w_h1t.as<float>(); g4.ldb = (int)ldt;
        g4.epi = EPI_STORE; g4.out = c->w_g4.as<float>(); g4.ldo = H;
        g4.split_stride = (size_t)H * H;
        RET(launch_gemm(c, g4, splits4, st));

        GemmArgs g5{};  // gW0 = D1^T X (split-K partials, 48 padded columns)
        g5.M = H; g5.N = 48; g5.K = nbr;
        g5.A = c->w_d1t.as<float>(); g5.lda = (int)ldt;
        g5.B = c->w_xt.as<float>(); g5.ldb = (int)ldt;
        g5.epi = EPI_STORE; g5.out = c->w_g5.as<float>(); g5.ldo = 48;
        g5.split_stride = (size_t)H * 48;
        RET(launch_gemm(c, g5, splits5, st));

        split_reduce_f32_kernel<<<blocks((size_t)H * H), 256, 0, st>>>(
            c->w_g4.as<float>(), splits4, (size_t)H * H, H, H, H, G + o_w1, H);
        RET(check_launch(c, "split_reduce_f32_kernel"));
        wide_gw0_kernel<<<blocks((size_t)H * (F + 1)), 256, 0, st>>>(c->w_g5.as<float>(), splits5,
                                                                     (size_t)H * 48, H, G, G + o_b0);
        RET(check_launch(c, "wide_gw0_kernel"));
        wide_head_reduce_kernel<<<(3 * H + 3 + 31) / 32, 256, 0, st>>>(
            c->w_part.as<double>(), (nbr + 31) / 32, H, G + o_w2, G + o_w2 + 2 * H, G + o_b1,
            c->w_loss.as<double>());
        RET(check_launch(c, "wide_head_reduce_kernel"));
    } else {
        CK(cudaMemsetAsync(G, 0, sizeof(float) * wide_param_count(H), st));
        CK(cudaMemsetAsync(c->w_loss.p, 0, sizeof(double), st));
    }
    if (c->comm) {
        CKN(ncclAllReduce(G, G, wide_param_count(H), ncclFloat32, ncclSum, c->comm, st));
        CKN(ncclAllReduce(c->w_loss.p, c->w_loss.p, 1, ncclFloat64, ncclSum, c->comm, st));
    }
    wide_update_kernel<<<blocks(wide_param_count(H)), 256, 0, st>>>(
        P, G, c->w_loss.as<double>(), nb, lr, H, c->w_w1t.as<float>(), c->w_w0p.as<float>(), epoch,
        c->diverged.as<int>(), c->epoch_acc.as<double>(), wide_param_count(H));
    return check_launch(c, "wide_update_kernel");
}

// ------------------------------------------------ BF16 path (k_wide16.cu)
// Launch with programmatic dependent launch: the kernel may start while its
// predecessor in the stream finishes (its griddepcontrol.wait orders the
// data); kept through stream capture as a programmatic graph edge.
template <typename... K, typename... A>
int launch_pdl_cl(gbxcu_ctx* c, const char* name, void (*kern)(K...), dim3 grid, dim3 block, size_t smem,
                  cudaStream_t st, dim3 cluster, A... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = cluster.x;
    at[1].val.clusterDim.y = cluster.y;
    at[1].val.clusterDim.z = cluster.z;
    cfg.attrs = at;
    cfg.numAttrs = cluster.x * cluster.y * cluster.z > 1 ? 2 : 1;
    CK(cudaLaunchKernelEx(&cfg, kern, args...));
    return check_launch(c, name);
}
template <typename... K, typename... A>
int launch_pdl(gbxcu_ctx* c, const char* name, void (*kern)(K...), dim3 grid, dim3 block, size_t smem,
               cudaStream_t st, A... args) {
    return launch_pdl_cl(c, name, kern, grid, block, smem, st, dim3(1, 1, 1), args...);
}

// K-major bf16 operand [rows][ld] (K valid columns) as TMA boxes of
// {64 bf16 = 128 B, box_rows} with the 128-byte swizzle; zero fill past K / rows.
bool make_bf16_map(CUtensorMap* m, const void* base, int K, int rows, int ld, int box_rows) {
    const EncodeTiledFn enc = encode_tiled();
    if (!enc) return false;
    const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
    const cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// bf16 epilogue output [rows][ld] (cols valid) as TMA store boxes of
// {box_cols, box_rows}, no swizzle; stores past cols / rows are clipped.
bool make_bf16_store_map(CUtensorMap* m, const void* base, int cols, int rows, int ld, int box_cols,
                         int box_rows) {
    const EncodeTiledFn enc = encode_tiled();
    if (!enc) return false;
    const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
    const cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// D = A B^T on the bf16 kernel: A [M][lda] (K valid), B [N][ldb]; grid (N/BN, M/128, splits).
// Epilogue outputs through TMA stores: g.out [M][g.ldo] row-major and g.out_t
// [N][g.ldt] transposed (each when non-null), in 32-row x 16-column chunks.
template <int BN, int ST, int EPI>
int launch_w16(gbxcu_ctx* c, const void* A, int lda, const void* B, int ldb, const W16Args& g, int splits,
               cudaStream_t st, int cluster_x = 1, int cluster_z = 1) {
    CUtensorMap ma, mb, mo{}, mot{};
    // (G3, EPI_D1T: B is MN-major — [K rows][N] — as {64 N, 64 K} boxes)
    const bool b_ok = EPI == W16_EPI_D1T ? make_bf16_map(&mb, B, g.N, g.K, ldb, 64)
                                         : make_bf16_map(&mb, B, g.K, g.N, ldb, BN > 256 ? 256 : BN);
    if (!make_bf16_map(&ma, A, g.K, g.M, lda, 128) || !b_ok)
        return fail(GBXCU_ECUDA, "cuTensorMapEncodeTiled unavailable or rejected a bf16 operand");
    if ((g.out && !make_bf16_store_map(&mo, g.out, g.N, g.M, g.ldo, 16, 32)) ||
        (g.out_t && !make_bf16_store_map(&mot, g.out_t, g.M, g.N, g.ldt, 32, 16)))
        return fail(GBXCU_ECUDA, "cuTensorMapEncodeTiled rejected a bf16 epilogue output");
    dim3 grid((g.N + BN - 1) / BN, (g.M + 127) / 128, splits);
    return launch_pdl_cl(c, "w16_gemm_kernel", w16_gemm_kernel<BN, ST, EPI>, grid,
                         dim3(128 * w_ew<EPI>()),
                         w16_gemm_smem_bytes<BN, ST>(), st, dim3(cluster_x, 1, cluster_z), ma, mb, mo, mot, g);
}

// The fused G4 + G5 + SGD launch: grid (1, T1 + T0, W16_SPLITS), clusters of
// W16_SPLITS along z; tiles y < T1 = (H/128)^2 are gW1 = D2^T H1 tiles, the
// T0 = H/128 others [gW0 | gb0] = D1^T [X | 1] tiles (maps in the o / ot slots).
// Operands are MN-major — the row-major D2 / H1 (gW1 tiles) and D1 / Xg (W0
// tiles), K = the records along their rows — as {64 M/N, 64 K} boxes, so no
// transposed copy of any activation is written on this path.
int launch_w16_sgd(gbxcu_ctx* c, const W16Args& g, const void* d1, const void* xg, cudaStream_t st) {
    const int H = g.M, K = g.K;
    CUtensorMap ma, mb, m5a, m5b;
    if (!make_bf16_map(&ma, c->b_d2.p, H, K, H, 64) || !make_bf16_map(&mb, c->b_h1.p, H, K, H, 64) ||
        !make_bf16_map(&m5a, d1, H, K, H, 64) || !make_bf16_map(&m5b, xg, 64, K, 64, 64))
        return fail(GBXCU_ECUDA, "cuTensorMapEncodeTiled unavailable or rejected a bf16 operand");
    const int nt = (H + 127) / 128;
    dim3 grid(1, nt * nt + nt, W16_SPLITS);
    return launch_pdl_cl(c, "w16_gemm_kernel", w16_gemm_kernel<128, 6, W16_EPI_SGD>, grid, dim3(512),
                         w16_gemm_smem_bytes<128, 6>(), st, dim3(1, 1, W16_SPLITS), ma, mb, m5a, m5b, g);
}

int check_hidden16(int H) {
    if (H < 64 || H > W16_MAX_H || H % 64 != 0)
        return fail(GBXCU_EINVAL, "bf16 wide MLP: hidden width must be a multiple of 64 in [64, 512]");
    return GBXCU_OK;
}

struct W16Plan {
    int H;
    size_t bmax, ldt;
    int s4, s5;
};

W16Plan w16_plan(gbxcu_ctx* c, int H, size_t bmax) {
    W16Plan P{H, bmax, (bmax + 7) & ~(size_t)7, 1, 1};
    // split-K so the K = batch GEMMs fill the machine
    const int kblocks = (int)((bmax + 63) / 64);
    const int tiles4 = ((H + 127) / 128) * ((H + 127) / 128), tiles5 = (H + 127) / 128;
    P.s4 = std::max(1, std::min(kblocks, c->num_sms / tiles4));
    P.s5 = std::max(1, std::min(kblocks, c->num_sms / tiles5));
    // no empty splits (each split covers ceil(kblocks / s) blocks)
    P.s4 = (kblocks + (kblocks + P.s4 - 1) / P.s4 - 1) / ((kblocks + P.s4 - 1) / P.s4);
    P.s5 = (kblocks + (kblocks + P.s5 - 1) / P.s5 - 1) / ((kblocks + P.s5 - 1) / P.s5);
    return P;
}

int w16_alloc(gbxcu_ctx* c, const W16Plan& P) {
    const size_t H = P.H, b = P.bmax, t = P.ldt, bf = 2;
    RET(c->b_xg.ensure(2 * bf * b * 64));  // (two copies: by step parity)
    RET(c->b_xt.ensure(2 * bf * 64 * t));
    RET(c->b_h1.ensure(bf * b * H));
    RET(c->b_h1t.ensure(bf * H * t));
    RET(c->b_d2.ensure(bf * b * H));
    RET(c->b_d2t.ensure(bf * H * t));
    RET(c->b_d1t.ensure(bf * H * t));
    RET(c->b_w0p.ensure(bf * H * 64));
    RET(c->b_w1.ensure(bf * H * H));
    RET(c->b_p4.ensure(sizeof(float) * (size_t)P.s4 * H * H));
    RET(c->b_p5.ensure(sizeof(float) * (size_t)P.s5 * H * 64));
    RET(c->b_hp.ensure(sizeof(double) * ((b + 127) / 128) * (3 * H + 3)));
    RET(c->w_grad.ensure(sizeof(float) * wide_param_count(P.H)));
    RET(c->w_loss.ensure(64));
    return GBXCU_OK;
}

// One SGD step on rows[0, nbr) (this rank's slice of a global batch of nb), BF16 path.
// timeline slot base of the step being enqueued (GBX_PHASE_TIMING builds)
int g_w16_dbg_step = -1;

// Xg / X^T live in two copies selected by the step's parity `par`: the next
// step's gather overwrites the other copy while this step's G4+G5 still
// reads X^T, so the gather runs beside it and waits for it only at its end.
int w16_step(gbxcu_ctx* c, const W16Plan& P, float* Pm, const float* feat, const double* tgt,
             const uint32_t* rows, int nbr, size_t nb, double lr, const int* epoch, cudaStream_t st, int par) {
#ifdef GBX_PHASE_TIMING
    const int dbg = g_w16_dbg_step >= 0 && g_w16_dbg_step < 8 ? 8 * g_w16_dbg_step : -100;
#else
    const int dbg = -100;
#endif
    auto slot = [&](int k) { return dbg >= 0 ? dbg + k : -1; };
    const int H = P.H, ldt = (int)P.ldt;
    const size_t o_b0 = (size_t)H * F, o_w1 = o_b0 + H, o_b1 = o_w1 + (size_t)H * H, o_w2 = o_b1 + H;
    using bf = __nv_bfloat16;
    bf* xg = c->b_xg.as<bf>() + (size_t)par * P.bmax * 64;
    bf* xt = c->b_xt.as<bf>() + (size_t)par * 64 * P.ldt;
    W16UpdArgs u{};
    u.params = Pm; u.hidden = H; u.np = wide_param_count(H); u.nb = nb; u.lr = lr;
    u.p4 = c->b_p4.as<float>(); u.s4 = P.s4; u.p5 = c->b_p5.as<float>(); u.s5 = P.s5;
    u.hp = c->b_hp.as<double>(); u.nhead = (nbr + 127) / 128;
    u.g_out = c->w_grad.as<float>(); u.loss_sum = c->w_loss.as<double>();
    u.w0p = c->b_w0p.as<bf>(); u.w1 = c->b_w1.as<bf>(); u.w1t = nullptr;  // (G3 reads W1 MN-major)
    u.epoch = epoch; u.diverged = c->diverged.as<int>(); u.epoch_acc = c->epoch_acc.as<double>();
    u.dbg = slot(6);
    if (nbr > 0) {
        RET(launch_pdl(c, "w16_gather_kernel", w16_gather_kernel, dim3((nbr + 63) / 64), dim3(256), 0, st, feat,
                       rows, nbr, dbg >= 0 ? slot(0) : -(g_w16_dbg_step + 2), xg, c->comm ? xt : nullptr, ldt));
        W16Args g1{};
        g1.dbg = slot(1);  // H1 = relu(Xg W0^T + b0) -> H1, H1^T
        g1.M = nbr; g1.N = H; g1.K = 64; g1.bias = Pm + o_b0;
        g1.out = c->b_h1.as<bf>(); g1.ldo = H; g1.out_t = c->comm ? c->b_h1t.as<bf>() : nullptr; g1.ldt = ldt;
        RET((launch_w16<256, 4, W16_EPI_H1>(c, xg, 64, c->b_w0p.p, 64, g1, 1, st)));
        W16Args g2{};
        g2.dbg = slot(2);  // acc = H1 W1^T -> fused head -> D2, D2^T, head partials
        g2.M = nbr; g2.N = H; g2.K = H; g2.bias = Pm + o_b1;
        g2.out = c->b_d2.as<bf>(); g2.ldo = H; g2.out_t = c->comm ? c->b_d2t.as<bf>() : nullptr; g2.ldt = ldt;
        g2.w2 = Pm + o_w2; g2.b2 = Pm + o_w2 + 2 * H; g2.tgt = tgt; g2.rows = rows;
        g2.inv_b = 1.0 / (double)nb; g2.head_part = c->b_hp.as<double>();
        // a CTA pair (cluster along x) per 128-row tile covers the full rows
        RET((launch_w16<256, 4, W16_EPI_HEAD>(c, c->b_h1.p, H, c->b_w1.p, H, g2, 1, st, (H + 255) / 256)));
        W16Args g3{};
        g3.dbg = slot(3);  // D1 = (D2 W1) [H1 > 0] -> D1^T
        g3.M = nbr; g3.N = H; g3.K = H; g3.mask = c->b_h1.as<bf>(); g3.ldm = H;
        if (c->comm) {  // D1^T for the split-K G5
            g3.out_t = c->b_d1t.as<bf>(); g3.ldt = ldt;
        } else {        // D1 row-major (same buffer) for the fused SGD launch
            g3.out = c->b_d1t.as<bf>(); g3.ldo = H;
        }
        RET((launch_w16<256, 4, W16_EPI_D1T>(c, c->b_d2.p, H, c->b_w1.p, H, g3, 1, st)));  // B = W1, MN-major
        W16Args g4{};
        g4.dbg = slot(4);  // gW1 = D2^T H1 (split-K partials)
        g4.M = H; g4.N = H; g4.K = nbr; g4.part = c->b_p4.as<float>(); g4.ldp = H;
        g4.split_stride = (size_t)H * H;
        W16Args g5{};
        g5.dbg = slot(5);  // gW0 | gb0 = D1^T [X | 1] (split-K partials)
        g5.M = H; g5.N = 64; g5.K = nbr; g5.part = c->b_p5.as<float>(); g5.ldp = 64;
        g5.split_stride = (size_t)H * 64;
        if (!c->comm) {
            // one rank: G4 and G5 share one launch whose epilogue reduces the
            // K splits across a cluster and applies SGD (no update launch)
            g4.u = u;
            g4.dbg = slot(4);
            return launch_w16_sgd(c, g4, c->b_d1t.p, xg, st);
        }
        RET((launch_w16<128, 6, W16_EPI_PART>(c, c->b_d2t.p, ldt, c->b_h1t.p, ldt, g4, P.s4, st)));
        RET((launch_w16<64, 6, W16_EPI_PART>(c, c->b_d1t.p, ldt, xt, ldt, g5, P.s5, st)));
    } else {
        // an empty slice contributes nothing (data-parallel remainder steps)
        CK(cudaMemsetAsync(c->b_p4.p, 0, sizeof(float) * (size_t)P.s4 * H * H, st));
        CK(cudaMemsetAsync(c->b_p5.p, 0, sizeof(float) * (size_t)P.s5 * H * 64, st));
        CK(cudaMemsetAsync(c->b_hp.p, 0, sizeof(double) * (3 * H + 3), st));
        u.nhead = 1;
    }
    int nb0, nw1, nb2;
    w16_update_layout(H, u.np, nb0, nw1, nb2);
    const int nblk = nb0 + nw1 + nb2;
    if (!c->comm) return launch_pdl(c, "w16_update_kernel", w16_update_kernel, dim3(nblk), dim3(256), 0, st, u, 0);
    w16_update_kernel<<<nblk, 256, 0, st>>>(u, 1);
    RET(check_launch(c, "w16_update_kernel"));
    CKN(ncclAllReduce(u.g_out, u.g_out, u.np, ncclFloat32, ncclSum, c->comm, st));
    CKN(ncclAllReduce(u.loss_sum, u.loss_sum, 1, ncclFloat64, ncclSum, c->comm, st));
    w16_update_kernel<<<nblk, 256, 0, st>>>(u, 2);
    return check_launch(c, "w16_update_kernel");
}

int w16_fit_device(gbxcu_ctx* c, int H, float* d_params, const float* d_feat, const double* d_tgt, size_t n,
                   const gbxcu_train_cfg* cfg, double* epoch_loss_out, int* diverged_epoch, cudaStream_t st) {
    RET(check_hidden16(H));
    RET(validate_cfg(cfg, n));
    if (cfg->loss_mode != GBXCU_LOSS_KL || cfg->optimizer != GBXCU_OPT_SGD)
        return fail(GBXCU_EINVAL, "the wide MLP trains with the reference's KL + SGD only");
    RET(setup_kernel_attrs());
    RET(prepare_order(c, n, st));
    const size_t b = std::min<size_t>((size_t)cfg->batch_size, n);
    const W16Plan P = w16_plan(c, H, (b + c->nranks - 1) / c->nranks);
    RET(w16_alloc(c, P));
    RET(c->epoch_loss.ensure(sizeof(double) * cfg->epochs));
    RET(c->epoch_acc.ensure(16));
    RET(c->w_epoch.ensure(16));
    using bf = __nv_bfloat16;
    w16_weights_kernel<<<blocks((size_t)H * H), 256, 0, st>>>(d_params, H, c->b_w0p.as<bf>(), c->b_w1.as<bf>(),
                                                              nullptr);
    RET(check_launch(c, "w16_weights_kernel"));
    const long n_steps = (long)((n + cfg->batch_size - 1) / cfg->batch_size);
    auto run_steps = [&](const uint32_t* order) -> int {
        for (long s = 0; s < n_steps; ++s) {
            const size_t start = (size_t)s * cfg->batch_size;
            const size_t nb = std::min(n, start + (size_t)cfg->batch_size) - start;
            const size_t per = (nb + c->nranks - 1) / c->nranks;
            const size_t lo = std::min(nb, (size_t)c->rank * per), hi = std::min(nb, lo + per);
            g_w16_dbg_step = (int)s;
            RET(w16_step(c, P, d_params, d_feat, d_tgt, order + start + lo, (int)(hi - lo), nb,
                         cfg->learning_rate, c->w_epoch.as<int>(), st, (int)(s & 1)));
        }
        return GBXCU_OK;
    };
    // an epoch's ~7 launches per step replay as a CUDA graph (single-GPU path)
    const char* ge = getenv("GBX_WIDE_GRAPH");
    const bool use_graph = !c->comm && n_steps > 1 && !(ge && ge[0] == '0');
    for (int e = 0; e < cfg->epochs; ++e) {
        RET(shuffle_epoch(c, n, cfg->seed, e, st));
        CK(cudaMemsetAsync(c->epoch_acc.p, 0, sizeof(double), st));
        CK(cudaMemcpyAsync(c->w_epoch.p, &e, sizeof(int), cudaMemcpyHostToDevice, st));
        const uint32_t* order = c->order.as<uint32_t>();
        if (!use_graph) {
            RET(run_steps(order));
        } else {
            double lr = cfg->learning_rate;
            uint64_t lr_bits;
            std::memcpy(&lr_bits, &lr, 8);
            const std::vector<const void*> key = {
                (const void*)(uintptr_t)16, order, d_params, d_feat, d_tgt, (const void*)(uintptr_t)H,
                (const void*)n, (const void*)(uintptr_t)cfg->batch_size, (const void*)(uintptr_t)lr_bits,
                (const void*)P.ldt, (const void*)(uintptr_t)P.s4, (const void*)(uintptr_t)P.s5,
                c->b_xg.p, c->b_xt.p, c->b_h1.p, c->b_h1t.p, c->b_d2.p, c->b_d2t.p, c->b_d1t.p,
                c->b_w0p.p, c->b_w1.p, c->b_p4.p, c->b_p5.p, c->b_hp.p, c->w_grad.p,
                c->w_loss.p, c->w_epoch.p, c->diverged.p, c->epoch_acc.p};
            gbxcu_ctx::WideGraph* g = nullptr;
            for (auto& x : c->wg)
                if (x.exec && x.key == key) g = &x;
            if (!g) {
                g = &c->wg[c->wg_next];
                c->wg_next ^= 1;
                if (g->exec) cudaGraphExecDestroy(g->exec);
                g->exec = nullptr;
                g->key.clear();
                if (getenv("GBX_DEBUG_GRAPH")) fprintf(stderr, "[gbxcu] capturing the wide-step graph\n");
                CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
                const int rc = run_steps(order);
                cudaGraph_t graph = nullptr;
                const cudaError_t ce = cudaStreamEndCapture(st, &graph);
                if (rc != GBXCU_OK) {
                    if (graph) cudaGraphDestroy(graph);
                    return rc;
                }
                if (ce != cudaSuccess) return fail(GBXCU_ECUDA, "wide-step graph capture failed");
                const cudaError_t ie = cudaGraphInstantiate(&g->exec, graph, 0);
                cudaGraphDestroy(graph);
                if (ie != cudaSuccess) {
                    g->exec = nullptr;
                    return fail(GBXCU_ECUDA, "wide-step graph instantiation failed");
                }
                g->key = key;
            }
            CK(cudaGraphLaunch(g->exec, st));
        }
        finish_epoch_kernel<<<1, 1, 0, st>>>(c->epoch_acc.as<double>(), n, e, c->diverged.as<int>(),
                                              c->epoch_loss.as<double>());
        RET(check_launch(c, "finish_epoch_kernel"));
    }
    int dv = -1;
    CK(cudaMemcpyAsync(&dv, c->diverged.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    if (epoch_loss_out)
        CK(cudaMemcpyAsync(epoch_loss_out, c->epoch_loss.p, sizeof(double) * cfg->epochs,
                           cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (diverged_epoch) *diverged_epoch = dv;
    if (dv >= 0)
        return fail(GBXCU_EDIVERGED, "training loss became non-finite at epoch " + std::to_string(dv));
    return GBXCU_OK;
}

int wide_fit_device(gbxcu_ctx* c, int H, float* d_params, const float* d_feat, const double* d_tgt,
                    size_t n, const gbxcu_train_cfg* cfg, double* epoch_loss_out,
                    int* diverged_epoch, cudaStream_t st) {
    RET(check_hidden(H));
    RET(validate_cfg(cfg, n));
    if (cfg->loss_mode != GBXCU_LOSS_KL || cfg->optimizer != GBXCU_OPT_SGD)
        return fail(GBXCU_EINVAL, "the wide MLP trains with the reference's KL + SGD only");
    RET(setup_kernel_attrs());
    RET(prepare_order(c, n, st));
    const size_t b = std::min<size_t>((size_t)cfg->batch_size, n);
    const size_t bmax = (b + c->nranks - 1) / c->nranks;
    const size_t ldt = (bmax + 3) & ~(size_t)3;
    // split-K so the two K = batch GEMMs fill the machine
    const int tiles4 = ((H + 127) / 128) * ((H + 127) / 128), tiles5 = (H + 127) / 128;
    const int kblocks = (int)((bmax + 31) / 32);
    const int splits4 = std::max(1, std::min(kblocks, c->num_sms / tiles4));
    const int splits5 = std::max(1, std::min(kblocks, c->num_sms / tiles5));
    const int rsplit = (int)std::max<size_t>(1, std::min<size_t>(64, bmax / 64));
    RET(wide_alloc(c, H, bmax, splits4, splits5, rsplit));
    RET(c->epoch_loss.ensure(sizeof(double) * cfg->epochs));
    RET(c->epoch_acc.ensure(16));
    wide_w1t_kernel<<<blocks((size_t)H * std::max(H, 48)), 256, 0, st>>>(d_params, H, c->w_w1t.as<float>(),
                                                                        c->w_w0p.as<float>());
    RET(check_launch(c, "wide_w1t_kernel"));
    const long n_steps = (long)((n + cfg->batch_size - 1) / cfg->batch_size);
    RET(c->w_epoch.ensure(16));
    auto run_steps = [&](const uint32_t* order) -> int {
        for (long s = 0; s < n_steps; ++s) {
            const size_t start = (size_t)s * cfg->batch_size;
            const size_t nb = std::min(n, start + (size_t)cfg->batch_size) - start;
            const size_t per = (nb + c->nranks - 1) / c->nranks;
            const size_t lo = std::min(nb, (size_t)c->rank * per), hi = std::min(nb, lo + per);
            RET(wide_step(c, H, d_params, d_feat, d_tgt, order + start + lo, (int)(hi - lo), nb, ldt,
                          cfg->learning_rate, c->w_epoch.as<int>(), splits4, splits5, rsplit, st));
        }
        return GBXCU_OK;
    };
    // one epoch = ~12 launches per step, most of them short: replay them as a
    // CUDA graph (single-GPU path; NCCL steps launch directly)
    const char* ge = getenv("GBX_WIDE_GRAPH");
    const bool use_graph = !c->comm && n_steps > 1 && !(ge && ge[0] == '0');
    for (int e = 0; e < cfg->epochs; ++e) {
        RET(shuffle_epoch(c, n, cfg->seed, e, st));
        CK(cudaMemsetAsync(c->epoch_acc.p, 0, sizeof(double), st));
        CK(cudaMemcpyAsync(c->w_epoch.p, &e, sizeof(int), cudaMemcpyHostToDevice, st));
        const uint32_t* order = c->order.as<uint32_t>();
        if (!use_graph) {
            RET(run_steps(order));
        } else {
            double lr = cfg->learning_rate;
            uint64_t lr_bits;
            std::memcpy(&lr_bits, &lr, 8);
            const std::vector<const void*> key = {
                order, d_params, d_feat, d_tgt, (const void*)(uintptr_t)H, (const void*)n,
                (const void*)(uintptr_t)cfg->batch_size, (const void*)(uintptr_t)lr_bits,
                (const void*)ldt, (const void*)(uintptr_t)splits4, (const void*)(uintptr_t)splits5,
                c->w_grad.p, c->w_w1t.p, c->w_h1.p, c->w_h2.p, c->w_d2.p, c->w_h1t.p, c->w_d2t.p,
                c->w_d1t.p, c->w_xt.p, c->w_xg.p, c->w_w0p.p, c->w_d3.p, c->w_kl.p, c->w_part.p,
                c->w_g4.p, c->w_g5.p, c->w_loss.p, c->w_epoch.p, c->diverged.p, c->epoch_acc.p};
            gbxcu_ctx::WideGraph* g = nullptr;
            for (auto& x : c->wg)
                if (x.exec && x.key == key) g = &x;
            if (!g) {
                g = &c->wg[c->wg_next];
                c->wg_next ^= 1;
                if (g->exec) cudaGraphExecDestroy(g->exec);
                g->exec = nullptr;
                g->key.clear();
                if (getenv("GBX_DEBUG_GRAPH")) fprintf(stderr, "[gbxcu] capturing the wide-step graph\n");
                CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
                const int rc = run_steps(order);
                cudaGraph_t graph = nullptr;
                const cudaError_t ce = cudaStreamEndCapture(st, &graph);
                if (rc != GBXCU_OK) {
                    if (graph) cudaGraphDestroy(graph);
                    return rc;
                }
                if (ce != cudaSuccess) return fail(GBXCU_ECUDA, "wide-step graph capture failed");
                const cudaError_t ie = cudaGraphInstantiate(&g->exec, graph, 0);
                cudaGraphDestroy(graph);
                if (ie != cudaSuccess) {
                    g->exec = nullptr;
                    return fail(GBXCU_ECUDA, "wide-step graph instantiation failed");
                }
                g->key = key;
            }
            CK(cudaGraphLaunch(g->exec, st));
        }
        finish_epoch_kernel<<<1, 1, 0, st>>>(c->epoch_acc.as<double>(), n, e, c->diverged.as<int>(),
                                              c->epoch_loss.as<double>());
        RET(check_launch(c, "finish_epoch_kernel"));
    }
    int dv = -1;
    CK(cudaMemcpyAsync(&dv, c->diverged.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    if (epoch_loss_out)
        CK(cudaMemcpyAsync(epoch_loss_out, c->epoch_loss.p, sizeof(double) * cfg->epochs,
                           cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (diverged_epoch) *diverged_epoch = dv;
    if (dv >= 0)
        return fail(GBXCU_EDIVERGED, "training loss became non-finite at epoch " + std::to_string(dv));
    return GBXCU_OK;
}

}  // namespace

extern "C" {

size_t gbxcu_wide_param_count(int hidden) { return wide_param_count(hidden); }

int gbxcu_wide_init(gbxcu_ctx* c, int hidden, uint64_t seed, float* params_out) {
    if (!c || !params_out) return fail(GBXCU_EINVAL, "null argument");
    RET(check_hidden(hidden));
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    const size_t np = wide_param_count(hidden);
    RET(c->w_params.ensure(sizeof(float) * np));
    wide_init_kernel<<<blocks(np), 256, 0, c->stream>>>(seed, hidden, c->w_params.as<float>(), np);
    RET(check_launch(c, "wide_init_kernel"));
    CK(cudaMemcpyAsync(params_out, c->w_params.p, sizeof(float) * np, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return GBXCU_OK;
}

int gbxcu_wide_forward(gbxcu_ctx* c, int hidden, const float* params, const float* feat, size_t n,
                       double* probs) {
    if (!c || !params || !probs || (n && !feat)) return fail(GBXCU_EINVAL, "null argument");
    RET(check_hidden(hidden));
    if (n == 0) return GBXCU_OK;
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    RET(setup_kernel_attrs());
    cudaStream_t st = c->stream;
    const int H = hidden;
    const size_t np = wide_param_count(H), chunk = std::min<size_t>(n, 65536);
    RET(upload(c->w_params, params, np, st));
    RET(upload(c->w_feat, feat, n * F, st));
    RET(c->w_probs.ensure(sizeof(double) * 2 * n));
    RET(c->w_h1.ensure(sizeof(float) * chunk * H));
    RET(c->w_h2.ensure(sizeof(float) * chunk * H));
    const float* P = c->w_params.as<float>();
    for (size_t r0 = 0; r0 < n; r0 += chunk) {
        const int m = (int)std::min(chunk, n - r0);
        GemmArgs g1{};
        g1.M = m; g1.N = H; g1.K = F;
        g1.A = c->w_feat.as<float>() + r0 * F; g1.lda = F;
        g1.B = P; g1.ldb = F;
        g1.epi = EPI_BIAS_RELU; g1.bias = P + (size_t)H * F;
        g1.out = c->w_h1.as<float>(); g1.ldo = H;
        RET(launch_gemm(c, g1, 1, st));
        GemmArgs g2{};
        g2.M = m; g2.N = H; g2.K = H;
        g2.A = c->w_h1.as<float>(); g2.lda = H;
        g2.B = P + (size_t)H * F + H; g2.ldb = H;
        g2.epi = EPI_BIAS_RELU; g2.bias = P + (size_t)H * F + H + (size_t)H * H;
        g2.out = c->w_h2.as<float>(); g2.ldo = H;
        RET(launch_gemm(c, g2, 1, st));
        const float* w2 = P + (size_t)H * F + H + (size_t)H * H + H;
        wide_probs_kernel<<<blocks((size_t)m * 32), 256, 0, st>>>(c->w_h2.as<float>(), w2, w2 + 2 * H, m,
                                                                  H, c->w_probs.as<double>() + 2 * r0);
        RET(check_launch(c, "wide_probs_kernel"));
    }
    CK(cudaMemcpyAsync(probs, c->w_probs.p, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return GBXCU_OK;
}

int gbxcu_wide_fit_ex(gbxcu_ctx* c, int hidden, int precision, float* params_inout, const float* feat,
                      const double* tgt, size_t n, const gbxcu_train_cfg* cfg, double* epoch_loss_out,
                      int* diverged_epoch) {
    if (!c || !params_inout || !feat || !tgt) return fail(GBXCU_EINVAL, "null argument");
    if (precision != GBXCU_WIDE_TF32 && precision != GBXCU_WIDE_BF16)
        return fail(GBXCU_EINVAL, "unknown wide-MLP precision");
    RET(precision == GBXCU_WIDE_BF16 ? check_hidden16(hidden) : check_hidden(hidden));
    RET(validate_cfg(cfg, n));
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    const size_t np = wide_param_count(hidden);
    RET(upload(c->w_params, params_inout, np, st));
    RET(upload(c->w_feat, feat, n * F, st));
    RET(upload(c->w_tgt, tgt, n * 2, st));
    int rc = precision == GBXCU_WIDE_BF16
                 ? w16_fit_device(c, hidden, c->w_params.as<float>(), c->w_feat.as<float>(),
                                  c->w_tgt.as<double>(), n, cfg, epoch_loss_out, diverged_epoch, st)
                 : wide_fit_device(c, hidden, c->w_params.as<float>(), c->w_feat.as<float>(),
                                   c->w_tgt.as<double>(), n, cfg, epoch_loss_out, diverged_epoch, st);
    if (rc != GBXCU_OK && rc != GBXCU_EDIVERGED) return rc;
    const std::string msg = g_err;
    CK(cudaMemcpyAsync(params_inout, c->w_params.p, sizeof(float) * np, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    g_err = msg;
    return rc;
}

int gbxcu_wide_fit(gbxcu_ctx* c, int hidden, float* params_inout, const float* feat, const double* tgt,
                   size_t n, const gbxcu_train_cfg* cfg, double* epoch_loss_out, int* diverged_epoch) {
    return gbxcu_wide_fit_ex(c, hidden, GBXCU_WIDE_TF32, params_inout, feat, tgt, n, cfg, epoch_loss_out,
                             diverged_epoch);
}

int gbxcu_wide_fit_ex_dev(gbxcu_ctx* c, int hidden, int precision, float* d_params, const float* d_feat,
                          const double* d_tgt, size_t n, const gbxcu_train_cfg* cfg, double* epoch_loss_out,
                          int* diverged_epoch, void* stream) {
    if (!c || !d_params || !d_feat || !d_tgt) return fail(GBXCU_EINVAL, "null argument");
    if (precision != GBXCU_WIDE_TF32 && precision != GBXCU_WIDE_BF16)
        return fail(GBXCU_EINVAL, "unknown wide-MLP precision");
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    if (precision == GBXCU_WIDE_BF16)
        return w16_fit_device(c, hidden, d_params, d_feat, d_tgt, n, cfg, epoch_loss_out, diverged_epoch,
                              pick(c, stream));
    return wide_fit_device(c, hidden, d_params, d_feat, d_tgt, n, cfg, epoch_loss_out, diverged_epoch,
                           pick(c, stream));
}

int gbxcu_wide_fit_dev(gbxcu_ctx* c, int hidden, float* d_params, const float* d_feat,
                       const double* d_tgt, size_t n, const gbxcu_train_cfg* cfg,
                       double* epoch_loss_out, int* diverged_epoch, void* stream) {
    return gbxcu_wide_fit_ex_dev(c, hidden, GBXCU_WIDE_TF32, d_params, d_feat, d_tgt, n, cfg,
                                 epoch_loss_out, diverged_epoch, stream);
}

// D[M][N] = bf16(A)[M][K] . bf16(B)[N][K]^T on the tcgen05 kind::f16 kernel
// (host fp32 buffers, rounded to bf16 on the device; fp32 result).
int gbxcu_bf16_gemm(gbxcu_ctx* c, int M, int N, int K, const float* A, const float* B, float* D) {
    if (!c || !A || !B || !D || M < 1 || N < 1 || K < 1) return fail(GBXCU_EINVAL, "bad gemm arguments");
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    RET(setup_kernel_attrs());
    cudaStream_t st = c->stream;
    const int ka = (K + 7) & ~7, np = (N + 15) & ~15;  // 16-B row strides; 16-column epilogue chunks
    std::vector<float> a((size_t)M * ka, 0.f), b((size_t)N * ka, 0.f);
    for (int r = 0; r < M; ++r) std::memcpy(&a[(size_t)r * ka], A + (size_t)r * K, sizeof(float) * K);
    for (int r = 0; r < N; ++r) std::memcpy(&b[(size_t)r * ka], B + (size_t)r * K, sizeof(float) * K);
    RET(upload(c->w_h1, a.data(), a.size(), st));
    RET(upload(c->w_h2, b.data(), b.size(), st));
    RET(c->b_h1.ensure(2 * a.size()));
    RET(c->b_d2.ensure(2 * b.size()));
    RET(c->w_d2.ensure(sizeof(float) * (size_t)M * np));
    to_bf16_kernel<<<blocks(a.size()), 256, 0, st>>>(c->w_h1.as<float>(), a.size(), c->b_h1.as<__nv_bfloat16>());
    to_bf16_kernel<<<blocks(b.size()), 256, 0, st>>>(c->w_h2.as<float>(), b.size(), c->b_d2.as<__nv_bfloat16>());
    RET(check_launch(c, "to_bf16_kernel"));
    W16Args g{};
    g.dbg = -1;
    g.M = M; g.N = N; g.K = K; g.part = c->w_d2.as<float>(); g.ldp = np; g.split_stride = 0;
    RET((launch_w16<256, 4, W16_EPI_PART>(c, c->b_h1.p, ka, c->b_d2.p, ka, g, 1, st)));
    std::vector<float> out((size_t)M * np);
    CK(cudaMemcpyAsync(out.data(), c->w_d2.p, sizeof(float) * out.size(), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int r = 0; r < M; ++r) std::memcpy(D + (size_t)r * N, &out[(size_t)r * np], sizeof(float) * N);
    return GBXCU_OK;
}

// Plain D[M][N] = A[M][K] . B[N][K]^T on the tcgen05 TF32 path (host buffers).
int gbxcu_tf32_gemm(gbxcu_ctx* c, int M, int N, int K, const float* A, const float* B, float* D) {
    if (!c || !A || !B || !D || M < 1 || N < 1 || K < 1) return fail(GBXCU_EINVAL, "bad gemm arguments");
    if (K % 4) return fail(GBXCU_EINVAL, "K must be a multiple of 4");
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    RET(setup_kernel_attrs());
    cudaStream_t st = c->stream;
    RET(upload(c->w_h1, A, (size_t)M * K, st));
    RET(upload(c->w_h2, B, (size_t)N * K, st));
    RET(c->w_d2.ensure(sizeof(float) * (size_t)M * N));
    GemmArgs g{};
    g.M = M; g.N = N; g.K = K;
    g.A = c->w_h1.as<float>(); g.lda = K;
    g.B = c->w_h2.as<float>(); g.ldb = K;
    g.epi = EPI_STORE; g.out = c->w_d2.as<float>(); g.ldo = N;
    RET(launch_gemm(c, g, 1, st));
    CK(cudaMemcpyAsync(D, c->w_d2.p, sizeof(float) * (size_t)M * N, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return GBXCU_OK;
}

}  // extern "C"
