// gbxcu_api.cu — the C ABI declared in include/gbxcu.h.
//
// Host-side orchestration only: argument validation (mirroring the
// reference's ValidationError cases), device buffers, launch configuration,
// the per-epoch shuffle -> train sequence of fit, and the NCCL all-reduce of
// the data-parallel step. All arithmetic on the path runs in the kernels; there
// is no CPU fallback.
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
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    int ensure(size_t bytes) {
        if (bytes <= cap) return GBXCU_OK;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        CK(cudaMalloc(&p, std::max<size_t>(bytes, 256)));
        cap = std::max<size_t>(bytes, 256);
        return GBXCU_OK;
    }
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
};

}  // namespace

struct gbxcu_ctx {
    int device = 0;
    int num_sms = 0;
    cudaStream_t stream = nullptr;
    uint64_t launches = 0;
    std::mutex mu;
    // scratch
    DevBuf params, feat, tgt, probs, actions, recheck, counters, flags;
    DevBuf order, order2, partials, red, bar, diverged, epoch_loss, epoch_acc;
    DevBuf sh_jp, sh_head, sh_nxt, sh_succ, sh_root, sh_root2, sh_flags;
    DevBuf seg_off, seg_seed, grad, scalar;
    DevBuf s_app_pipe, s_pipe_slot, s_slot_shader, s_slot_frac, s_pipe_wt, s_shader_lat, s_app_f64;
    DevBuf s_actions, s_run_seed, s_rows, s_samples, h_lower, h_count, h_nbins;
    int shuffle_grid = 0;
    int fast_per_sm = 1;
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
        set((const void*)train_epoch_kernel<32>, train_smem_bytes(32));
        set((const void*)train_epoch_kernel<64>, train_smem_bytes(64));
        set((const void*)train_partial_kernel<32>, train_smem_bytes(32));
        set((const void*)train_partial_kernel<64>, train_smem_bytes(64));
        set((const void*)batch_grad_kernel, train_smem_bytes(64));
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
                DevBuf& recheck, DevBuf& counters, DevBuf& flags) {
    if (n == 0) return GBXCU_OK;
    if (n > 0xFFFFFFFFull) return fail(GBXCU_EINVAL, "batch too large (> 2^32 states)");
    const int bits = (d_probs ? FWD_PROBS : 0) | (d_actions ? FWD_ACTIONS : 0) |
                     (d_seg_off ? FWD_COLLECT : 0);
    RET(counters.ensure(16));
    RET(flags.ensure(16));
    CK(cudaMemsetAsync(counters.p, 0, 16, st));
    CK(cudaMemsetAsync(flags.p, 0, 16, st));
    if (mode == GBXCU_FWD_FAST) {
        RET(recheck.ensure(n * sizeof(uint32_t)));
        const size_t warps = (n + 31) / 32;
        const size_t blocks_needed = (warps + FWD_BLOCK / 32 - 1) / (FWD_BLOCK / 32);
        const int grid = (int)std::min<size_t>(blocks_needed, (size_t)c->num_sms * c->fast_per_sm);
        fwd_fast_kernel<<<grid, FWD_BLOCK, fast_smem_bytes(), st>>>(
            d_params, d_feat, n, d_probs, d_actions, d_seg_off, nseg, d_seg_seed, eps,
            recheck.as<uint32_t>(), counters.as<unsigned int>(), flags.as<unsigned int>(), bits);
        RET(check_launch(c, "fwd_fast_kernel"));
        fwd_exact_kernel<<<c->num_sms * 2, EXACT_BLOCK, exact_smem_bytes(), st>>>(
            d_params, d_feat, n, recheck.as<uint32_t>(), counters.as<unsigned int>(), d_probs,
            d_actions, d_seg_off, nseg, d_seg_seed, eps, flags.as<unsigned int>(), bits);
        RET(check_launch(c, "fwd_exact_kernel(recheck)"));
    } else {
        const size_t blocks_needed = (n + EXACT_BLOCK - 1) / EXACT_BLOCK;
        const int grid = (int)std::min<size_t>(blocks_needed, (size_t)c->num_sms * 8);
        fwd_exact_kernel<<<grid, EXACT_BLOCK, exact_smem_bytes(), st>>>(
            d_params, d_feat, n, nullptr, nullptr, d_probs, d_actions, d_seg_off, nseg,
            d_seg_seed, eps, flags.as<unsigned int>(), bits);
        RET(check_launch(c, "fwd_exact_kernel"));
    }
    return GBXCU_OK;
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
    return GBXCU_OK;
}

// CTAs per step and records per tile: spread each rank's share of the batch
// over up to one CTA per SM in tiles of 32 records; switch to 64-record
// tiles once every SM already has more than 32 records.
void train_grid(gbxcu_ctx* c, const gbxcu_train_cfg* cfg, size_t n, int& G, int& tb) {
    const size_t b = std::min<size_t>((size_t)cfg->batch_size, n);
    const size_t per_rank = (b + c->nranks - 1) / c->nranks;
    G = (int)std::min<size_t>((per_rank + 31) / 32, (size_t)c->num_sms);
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
    RET(c->bar.ensure(16));
    RET(c->diverged.ensure(16));
    CK(cudaMemsetAsync(c->diverged.p, 0xFF, 16, st));
    iota_kernel<<<std::max(1, std::min<int>((int)((n + 255) / 256), c->num_sms * 8)), 256, 0, st>>>(
        c->order.as<uint32_t>(), n);
    return check_launch(c, "iota_kernel");
}

int fit_device(gbxcu_ctx* c, float* d_params, const float* d_feat, const double* d_tgt, size_t n,
               const gbxcu_train_cfg* cfg, double* epoch_loss_out, int* diverged_epoch,
               cudaStream_t st) {
    RET(validate_cfg(cfg, n));
    RET(setup_kernel_attrs());
    RET(prepare_order(c, n, st));
    RET(c->epoch_loss.ensure(sizeof(double) * cfg->epochs));
    RET(c->epoch_acc.ensure(16));
    int G = 1, tb = 32;
    train_grid(c, cfg, n, G, tb);
    RET(c->partials.ensure(sizeof(double) * (size_t)G * (NP + 1)));
    RET(c->red.ensure(sizeof(double) * (NP + 1)));

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
    const long n_steps = (long)((n + cfg->batch_size - 1) / cfg->batch_size);

    for (int e = 0; e < cfg->epochs; ++e) {
        RET(shuffle_epoch(c, n, cfg->seed, e, st));
        a.order = c->order.as<uint32_t>();  // the pass output (buffers ping-pong)
        a.epoch = e;
        if (!c->comm) {
            CK(cudaMemsetAsync(c->bar.as<unsigned int>() + 2, 0, 8, st));
            void* args[] = {&a};
            const void* fn = tb == 32 ? (const void*)train_epoch_kernel<32>
                                      : (const void*)train_epoch_kernel<64>;
            if (G == 1) {
                CK(cudaLaunchKernel(fn, 1, TRAIN_BLOCK, args, train_smem_bytes(tb), st));
            } else {
                CK(cudaLaunchCooperativeKernel(fn, G, TRAIN_BLOCK, args, train_smem_bytes(tb), st));
            }
            RET(check_launch(c, "train_epoch_kernel"));
        } else {
            CK(cudaMemsetAsync(c->epoch_acc.p, 0, sizeof(double), st));
            for (long s = 0; s < n_steps; ++s) {
                const size_t start = (size_t)s * cfg->batch_size;
                const size_t nb = std::min(n, start + (size_t)cfg->batch_size) - start;
                if (tb == 32)
                    train_partial_kernel<32><<<G, TRAIN_BLOCK, train_smem_bytes(32), st>>>(a, s);
                else
                    train_partial_kernel<64><<<G, TRAIN_BLOCK, train_smem_bytes(64), st>>>(a, s);
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
    int dv = -1;
    CK(cudaMemcpyAsync(&dv, c->diverged.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    if (epoch_loss_out)
        CK(cudaMemcpyAsync(epoch_loss_out, c->epoch_loss.p, sizeof(double) * cfg->epochs,
                           cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (diverged_epoch) *diverged_epoch = dv;
    if (dv >= 0)
        return fail(GBXCU_EDIVERGED,
                    "training loss became non-finite at epoch " + std::to_string(dv));
    return GBXCU_OK;
}

template <typename T>
int upload(DevBuf& b, const T* host, size_t count, cudaStream_t st) {
    RET(b.ensure(sizeof(T) * count));
    if (count) CK(cudaMemcpyAsync(b.p, host, sizeof(T) * count, cudaMemcpyHostToDevice, st));
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
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
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
    *out = c;
    return GBXCU_OK;
}

void gbxcu_destroy(gbxcu_ctx* c) {
    if (!c) return;
    if (c->comm) ncclCommDestroy(c->comm);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

void* gbxcu_stream(gbxcu_ctx* c) { return c ? (void*)c->stream : nullptr; }
uint64_t gbxcu_launch_count(const gbxcu_ctx* c) { return c ? c->launches : 0; }

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
    RET(upload(c->params, params_inout, NP, st));
    RET(upload(c->feat, feat, n * F, st));
    RET(upload(c->tgt, tgt, n * 2, st));
    int rc = fit_device(c, c->params.as<float>(), c->feat.as<float>(), c->tgt.as<double>(), n, cfg,
                        epoch_loss_out, diverged_epoch, st);
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

int gbxcu_comm_destroy(gbxcu_ctx* c) {
    if (!c) return fail(GBXCU_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(c->mu);
    if (c->comm) CKN(ncclCommDestroy(c->comm));
    c->comm = nullptr;
    c->nranks = 1;
    c->rank = 0;
    return GBXCU_OK;
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
    const int grid = (int)std::min<size_t>((s->n_apps + 7) / 8, (size_t)c->num_sms * 8);
    aggregate_kernel<<<grid, AGG_BLOCK, 0, st>>>(a);
    RET(check_launch(c, "aggregate_kernel"));
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
    RET(run_forward(c, d_params, s->features.as<float>(), s->n_shaders, nullptr, d_actions,
                    GBXCU_FWD_FAST, nullptr, 0, nullptr, 0.0, st, recheck, counters, flags));
    if (s->n_apps == 0) return GBXCU_OK;
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
    const int grid = (int)std::min<size_t>((s->n_apps + 7) / 8, (size_t)c->num_sms * 8);
    aggregate_kernel<<<grid, AGG_BLOCK, 0, st>>>(a);
    return check_launch(c, "aggregate_kernel");
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
