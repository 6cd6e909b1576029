/*
 * gbxcu.h — C ABI of the B200 (sm_100a) implementation of the gbxtune hot path.
 *
 * The reference (arXiv 2111.12055 analog, /root/reference/proj) exposes the
 * path only as C++ functions of the static library `gbx`; it has no FFI or
 * plugin registry. Each entry point below replaces one of those functions
 * (cited per declaration) with a batched, device-executed equivalent. The C++
 * drop-in mirror (headers under paper_2111_12055_b200/include/gbx/) and the Python
 * binding (paper_2111_12055_b200/__init__.py, ctypes) both bind exactly this
 * surface; INTEGRATION.md shows the binding a maintainer adds.
 *
 * Conventions
 *   - Plain pointers and sizes only; no C++ or torch types cross the ABI.
 *   - Functions without a `_dev` suffix take caller-owned HOST buffers and are
 *     synchronous. `_dev` variants take DEVICE pointers plus a cudaStream_t
 *     (passed as void*, NULL = the context's stream) and are asynchronous
 *     unless noted.
 *   - Parameters are the 5,026 fp32 values of the 44->64->32->2 policy in the
 *     reference's flat serialization order (proj/src/policy.cpp:152-182):
 *     w0[64][44] b0[64] w1[32][64] b1[32] w2[2][32] b2[2].
 *   - Features: [n][44] fp32 rows (176 B). Targets: [n][2] fp64.
 *   - Actions: uint8, 0 = Wave32, 1 = Wave64 (proj/include/gbx/core.hpp:19).
 *   - Every call returns a gbxcu_status. On failure gbxcu_last_error() holds
 *     a message. There is no CPU fallback: without a usable sm_100 device every
 *     compute entry point fails with GBXCU_ECUDA.
 */
#ifndef GBXCU_H
#define GBXCU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GBXCU_ABI_VERSION 2

#define GBXCU_N_FEATURES 44
#define GBXCU_N_PARAMS 5026

typedef enum {
    GBXCU_OK = 0,
    GBXCU_EINVAL = 1,      /* ValidationError (bad config, empty dataset, ...) */
    GBXCU_EDIVERGED = 2,   /* TrainingDivergedError; epoch reported separately */
    GBXCU_ECUDA = 3,       /* CUDA runtime / launch failure, or no device */
    GBXCU_ENCCL = 4,       /* NCCL failure in the data-parallel path */
    GBXCU_ENONFINITE = 5,  /* ValidationError: non-finite feature in forward */
    GBXCU_ETEMPERATURE = 6, /* InvalidTemperatureError (rho <= 0) */
    GBXCU_ECLOCK = 7        /* ClockRegressionError (q_update before the entry timestamp) */
} gbxcu_status;

/* Inference precision.
 *   EXACT: fp64 forward in the reference's summation order (bias first,
 *          ascending index, no FMA contraction where products round); probs
 *          match PolicyNet::forward to the last ulp of exp().
 *   FAST : fp32 forward + a rigorous per-state error bound; every state whose
 *          logit margin is inside the bound is re-run in EXACT mode, so the
 *          ACTIONS are identical to EXACT; probabilities are fp32-accurate
 *          (relative error <= 1e-5). */
typedef enum { GBXCU_FWD_EXACT = 0, GBXCU_FWD_FAST = 1 } gbxcu_fwd_mode;

typedef struct gbxcu_ctx gbxcu_ctx;

/* ----------------------------------------------------------------- context */
int gbxcu_abi_version(void);
const char* gbxcu_last_error(void); /* thread-local message of the last failure */
int gbxcu_create(int device, gbxcu_ctx** out);
void gbxcu_destroy(gbxcu_ctx* ctx);
/* cudaStream_t the context enqueues on when a _dev call passes NULL. */
void* gbxcu_stream(gbxcu_ctx* ctx);
/* Number of kernels this context launched since creation (for bench.py's
 * gpu_launches claim; counts our kernels only, not memcpys or NCCL). */
uint64_t gbxcu_launch_count(const gbxcu_ctx* ctx);
/* Device time (CUDA events on the launching stream) of the last single-GPU
 * fit with <= 8 epochs: epoch-permutation replay and train_epoch kernel,
 * summed over epochs (0 for the data-parallel path). */
int gbxcu_last_fit_timing(const gbxcu_ctx* ctx, double* shuffle_ms, double* train_kernel_ms);
/* Device time (CUDA events on the call's stream) of the last gbxcu_evaluate[_dev]
 * on this context: the inference (fast forward + exact re-check) and the
 * per-app aggregation (frame_time / run_benchmark rows). Waits for that call. */
int gbxcu_last_eval_timing(gbxcu_ctx* ctx, double* infer_ms, double* aggregate_ms);
/* States the last FAST-mode gbxcu_forward[_dev] on this context sent to the
 * exact fp64 re-check (guard margin inside the fp32 error bound). Synchronises
 * the device. */
int gbxcu_last_recheck_count(gbxcu_ctx* ctx, uint64_t* count);

/* ------------------------------------------------------------------- init */
/* PolicyNet::init (proj/src/policy.cpp:128-139) computed on the device:
 * fan-scaled uniform weights from derive_seed({seed,0x1A17,l}), zero biases. */
int gbxcu_policy_init(gbxcu_ctx* ctx, uint64_t seed, float* params_out);

/* -------------------------------------------------------------- inference */
/* PolicyNet::forward + select_greedy, batched (proj/src/policy.cpp:141-148,
 * 339-342). probs [n][2] and actions [n] are each nullable. Non-finite
 * features -> GBXCU_ENONFINITE (the whole call fails, like the first throwing
 * forward() in a reference loop). */
int gbxcu_forward(gbxcu_ctx* ctx, const float* params, const float* feat, size_t n,
                  double* probs, uint8_t* actions, int mode);
int gbxcu_forward_dev(gbxcu_ctx* ctx, const float* d_params, const float* d_feat, size_t n,
                      double* d_probs, uint8_t* d_actions, int mode, void* stream);

/* select_greedy over a batch (SURVEY §8b's gbxcu_forward_batch): FAST mode of
 * gbxcu_forward — actions exact, probabilities fp32-accurate. */
int gbxcu_forward_batch(gbxcu_ctx* ctx, const float* params, const float* feat, size_t n,
                        double* probs, uint8_t* actions);
/* select_sample (proj/src/policy.cpp:344-347) over a batch drawing from ONE
 * SplitMix64 stream whose current state is rng_state: state j takes the
 * stream's (j+1)-th next_unit(), Wave32 iff it is < p0. Exact decisions; the
 * caller's stream advances by n draws (SplitMix64::discard(n) in gbx/rng.hpp). */
int gbxcu_sample_batch(gbxcu_ctx* ctx, const float* params, const float* feat, size_t n,
                       uint64_t rng_state, uint8_t* actions);

/* Sampled (collection) decisions, proj/src/tuner.cpp:183-196 with
 * select_sample semantics (proj/src/policy.cpp:344-347): states are grouped
 * in segments (one per benchmark, seg_off[nseg+1]); segment b draws from
 * SplitMix64(seg_seed[b]) two uniforms per state (u_explore, u_action) in
 * state order; u_explore < eps -> Wave32 iff u_action < 0.5, else Wave32 iff
 * u_action < p0. Decisions are exact (fp64 re-check inside the margin). */
int gbxcu_collect(gbxcu_ctx* ctx, const float* params, const float* feat,
                  const uint64_t* seg_off, size_t nseg, const uint64_t* seg_seed, double eps,
                  uint8_t* actions);
int gbxcu_collect_dev(gbxcu_ctx* ctx, const float* d_params, const float* d_feat,
                      const uint64_t* d_seg_off, size_t nseg, const uint64_t* d_seg_seed,
                      size_t n_states, double eps, uint8_t* d_actions, void* stream);

/* ------------------------------------------------------- loss / gradient */
/* batch_kl_loss (proj/src/policy.cpp:194-201). */
int gbxcu_batch_kl_loss(gbxcu_ctx* ctx, const float* params, const float* feat,
                        const double* tgt, size_t n, double* loss_out);
/* batch_kl_gradient (proj/src/policy.cpp:270-279): grad_out[5026] fp64, flat
 * order; record contributions summed in batch order (bit-exact up to log()). */
int gbxcu_batch_kl_gradient(gbxcu_ctx* ctx, const float* params, const float* feat,
                            const double* tgt, size_t n, double* grad_out);

/* -------------------------------------------------------------------- fit */
typedef struct {
    double learning_rate; /* TrainConfig::learning_rate (> 0) */
    int epochs;           /* >= 1 */
    int batch_size;       /* >= 1; global batch across all ranks */
    uint64_t seed;        /* TrainConfig::seed (epoch shuffle stream) */
    int max_ctas;         /* 0 = auto (1 CTA per 32 records of the per-rank batch, <= #SMs) */
    int virtual_ranks;    /* 0/1 = off. V in 2..8: run the fused peer-set path with V ranks
                             inside one launch on this GPU (tests of the multi-GPU kernel) */
    /* Variants the north star names and the reference lacks ("parity unpinned";
     * restated in oracle/gbx_oracle.c:orc_fit_variant). Zero = the reference. */
    int loss_mode;        /* GBXCU_LOSS_KL (fit's distillation) | GBXCU_LOSS_TD: regression of
                             the taken action's output Q(x,a) on the reward, records
                             tgt[r] = {a (0/1), r}: L = mean (Q(x,a) - r)^2 */
    int optimizer;        /* GBXCU_OPT_SGD (fit's update) | GBXCU_OPT_ADAM (fp64 moments, owned
                             by the reducing CTA of each parameter slice) */
    double adam_beta1, adam_beta2, adam_eps;  /* 0 -> 0.9, 0.999, 1e-8 */
} gbxcu_train_cfg;
#define GBXCU_LOSS_KL 0
#define GBXCU_LOSS_TD 1
#define GBXCU_OPT_SGD 0
#define GBXCU_OPT_ADAM 1

/* fit (proj/src/policy.cpp:297-337): seeded in-place Fisher-Yates per epoch
 * (reproduced on the device), minibatch KL loss, analytic gradient, SGD
 * w = float(double(w) - lr*g). params_inout is updated in place; on
 * GBXCU_EDIVERGED it holds the last successful update and *diverged_epoch is
 * set (TrainingDivergedError semantics). epoch_loss_out[epochs] nullable.
 * With a communicator attached (gbxcu_comm_init) every global batch is split
 * into equal contiguous slices per rank and the flat fp64 gradient (+ loss)
 * is all-reduced once per step; all ranks must pass identical arguments. */
int gbxcu_fit(gbxcu_ctx* ctx, float* params_inout, const float* feat, const double* tgt, size_t n,
              const gbxcu_train_cfg* cfg, double* epoch_loss_out, int* diverged_epoch);
/* Device-resident form: d_params updated in place on the device; the epoch
 * losses are copied to the host buffer at the end (synchronous). */
int gbxcu_fit_dev(gbxcu_ctx* ctx, float* d_params, const float* d_feat, const double* d_tgt,
                  size_t n, const gbxcu_train_cfg* cfg, double* epoch_loss_out,
                  int* diverged_epoch, void* stream);

/* Permutation `order` after `epochs` Fisher-Yates passes of fit (device
 * deterministic-reservations replay of proj/src/policy.cpp:303-314). */
int gbxcu_fit_order(gbxcu_ctx* ctx, size_t n, uint64_t seed, int epochs, uint32_t* order_out);

/* -------------------------------------------------- data-parallel plumbing */
#define GBXCU_COMM_ID_BYTES 128
int gbxcu_comm_unique_id(uint8_t id_out[GBXCU_COMM_ID_BYTES]);
int gbxcu_comm_init(gbxcu_ctx* ctx, const uint8_t id[GBXCU_COMM_ID_BYTES], int nranks, int rank);
int gbxcu_comm_destroy(gbxcu_ctx* ctx);

/* Fused data-parallel path over NVLink peer memory (one process per GPU).
 * Instead of a per-step NCCL all-reduce, the multi-CTA train kernel of every
 * rank exchanges gradient partials, arrival counts and the updated
 * parameters directly in the peers' memory (reduce-scatter over all ranks'
 * CTAs, then an LL-word all-gather) — one launch per epoch on every GPU.
 * Protocol: every rank calls gbxcu_peer_export, the 64-byte handles are
 * all-gathered by the caller (e.g. torch.distributed), every rank calls
 * gbxcu_peer_attach with all of them, then the caller barriers before the
 * first fit. All ranks must then make identical fit calls (as with NCCL).
 * Replaces the all-reduce of the gradient in fit (proj/src/policy.cpp:327-332
 * run data-parallel; the reference itself is single-threaded). */
#define GBXCU_PEER_HANDLE_BYTES 64
int gbxcu_peer_export(gbxcu_ctx* ctx, uint8_t handle_out[GBXCU_PEER_HANDLE_BYTES]);
int gbxcu_peer_attach(gbxcu_ctx* ctx, int nranks, int rank, const uint8_t* handles);
int gbxcu_peer_detach(gbxcu_ctx* ctx);

/* ------------------------------------------------- experience store (Q-table) */
/* Device-resident QTable (proj/include/gbx/qtable.hpp:53-100): unique
 * StateKeys (30 u32, lexicographic order) with an optional {q, last check-in,
 * update count} per action. Hyper-parameters validated like
 * QHyperparams::validate (GBXCU_EINVAL). */
typedef struct gbxcu_qtable gbxcu_qtable;
#define GBXCU_KEY_WORDS 30
int gbxcu_qtable_create(gbxcu_ctx* ctx, double alpha, double omega, gbxcu_qtable** out);
void gbxcu_qtable_free(gbxcu_qtable* t);
int gbxcu_qtable_clear(gbxcu_qtable* t);  /* empty table, device buffers kept */
/* QTable::update (proj/src/qtable.cpp:76-92) applied to n tuples in order:
 * keys[n][30], actions[n] (0/1), rewards[n], now[n]. Same-key updates fold
 * sequentially (bit-exact for omega == 1, the reference default; pow() within
 * an ulp otherwise). GBXCU_ECLOCK at the first tuple whose check-in precedes
 * its entry's timestamp: *bad_index = that tuple, and the table holds exactly
 * the updates before it (as the reference does after the throw). */
int gbxcu_qtable_update_batch(gbxcu_qtable* t, const uint32_t* keys, const uint8_t* actions,
                              const double* rewards, const uint64_t* now, size_t n,
                              size_t* bad_index);
/* Device-resident tuples (actions must be 0/1; not re-validated). */
int gbxcu_qtable_update_batch_dev(gbxcu_qtable* t, const uint32_t* d_keys, const uint8_t* d_actions,
                                  const double* d_rewards, const uint64_t* d_now, size_t n,
                                  size_t* bad_index);
int gbxcu_qtable_size(const gbxcu_qtable* t, size_t* states, size_t* entries);
/* Replace the table with m states in key order (keys strictly increasing,
 * else GBXCU_EINVAL) — e.g. a table read by QTable::load (qtable.cpp:188-231). */
int gbxcu_qtable_import(gbxcu_qtable* t, const uint32_t* keys, const double* q, const uint64_t* ts,
                        const uint64_t* cnt, const uint8_t* has, size_t m);
/* Table in key order: keys[m][30], q/ts/cnt/has[m][2] (has: entry recorded). */
int gbxcu_qtable_export(const gbxcu_qtable* t, uint32_t* keys, double* q, uint64_t* ts,
                        uint64_t* cnt, uint8_t* has);
/* Binary columnar table file — the experience-store load path without text
 * parsing (the text form stays QTable::save / QTable::load,
 * proj/src/qtable.cpp:160-231). Little-endian; a 64-byte header
 * ("GBXQTAB", version 1, key words 30, states m, alpha, omega, payload bytes,
 * FNV-1a-64 checksum of the payload) then 64-byte-aligned columns keys[m][30]
 * u32 | q[m][2] f64 | t[m][2] u64 | count[m][2] u64 | has[m][2] u8, keys in
 * strictly increasing order. Load replaces the table and its alpha/omega
 * (as QTable::load does); GBXCU_EINVAL on a bad magic/version/size/checksum,
 * unsorted keys or an entry with zero updates. */
int gbxcu_qtable_save_columnar(const gbxcu_qtable* t, const char* path);
int gbxcu_qtable_load_columnar(gbxcu_qtable* t, const char* path);
/* snapshot_policy_dataset (proj/src/qtable.cpp:143-155): one record per key
 * with both actions, key order; feat[rows][44] = encode_state(counters_from_key)
 * (bit-exact: glibc log1pf restated), tgt[rows][2] = boltzmann_pair (CUDA exp:
 * within 2 ulp). feat == NULL: *rows only. GBXCU_ETEMPERATURE if rho <= 0. */
int gbxcu_qtable_snapshot(gbxcu_qtable* t, double rho, float* feat, double* tgt, size_t cap,
                          size_t* rows);
/* Device-resident form: writes straight into fit's input buffers. */
int gbxcu_qtable_snapshot_dev(gbxcu_qtable* t, double rho, float* d_feat, double* d_tgt, size_t cap,
                              size_t* rows);

/* ------------------------------------------------------------ aggregation */
/* Application suite in CSR form (the per-benchmark data SimSuite::frame_time
 * reads, proj/src/simenv.cpp:439-474; proj/include/gbx/simenv.hpp:55-100).
 * App (benchmark) ids are their indices. */
typedef struct {
    size_t n_apps, n_pipes, n_slots, n_shaders;
    const uint64_t* app_pipe_off;  /* [n_apps+1]  pipelines of app a          */
    const uint64_t* pipe_slot_off; /* [n_pipes+1] slots of pipeline p          */
    const uint32_t* slot_shader;   /* [n_slots]   shader id                    */
    const double* slot_frac;       /* [n_slots]   exec_fraction                */
    const double* pipe_wt;         /* [n_pipes][2] weight, base_time (s)       */
    const double* shader_lat;      /* [n_shaders][3] divergence, bandwidth_demand, parallelism */
    const double* app_f64;         /* [n_apps][4] baseline_fps, bandwidth_capacity (+inf =
                                       unconstrained), noise_sigma, memory_bound_threshold */
} gbxcu_suite;

/* Per-app frame time + noisy samples + reward/uplift for a per-shader action
 * vector: run_benchmark (proj/src/simenv.cpp:481-510), attribute_rewards /
 * reward_from_framerate (proj/src/tuner.cpp:131-147, core.cpp:125-133) and
 * evaluate's uplift (proj/src/tuner.cpp:282-289). run_seed[a] is the seed the
 * caller hands run_benchmark for app a. rows_out [n_apps][5] =
 * frame_time, true_fps, mean sample fps, uplift_pct, reward. samples_out
 * [n_apps][n_samples] nullable. Bit-exact vs the reference. */
int gbxcu_aggregate(gbxcu_ctx* ctx, const gbxcu_suite* suite, const uint8_t* shader_actions,
                    const uint64_t* run_seed, int n_samples, double* rows_out,
                    double* samples_out);

/* evaluate's 1%-bin histogram (proj/src/tuner.cpp:293-313). Writes up to
 * cap bins; *n_bins = the true bin count. */
int gbxcu_histogram(gbxcu_ctx* ctx, const double* uplift, size_t n, double* lower_out,
                    uint64_t* count_out, size_t cap, size_t* n_bins);

/* Device-resident suite handle (uploaded once, reused per sweep). The suite
 * arrays and features may live in host or device memory (unified addressing). */
typedef struct gbxcu_dsuite gbxcu_dsuite;
int gbxcu_suite_upload(gbxcu_ctx* ctx, const gbxcu_suite* host, const float* shader_features,
                       gbxcu_dsuite** out);
void gbxcu_suite_free(gbxcu_dsuite* s);
/* Raw device pointers of an uploaded suite (features [n_shaders][44] fp32). */
const float* gbxcu_suite_features(const gbxcu_dsuite* s);

/* One app-range shard of evaluate (multi-GPU: each rank evaluates
 * [app_lo, app_hi) of the same uploaded suite, inferring only the shaders
 * those apps reference; seeds use global app indices, so the gathered rows
 * equal gbxcu_evaluate's bit for bit and the histogram is built once from
 * them — SURVEY §8e). rows_out [app_hi - app_lo][5]. */
int gbxcu_evaluate_shard(gbxcu_ctx* ctx, const gbxcu_dsuite* suite, const float* params,
                         int n_samples, uint64_t seed, size_t app_lo, size_t app_hi,
                         double* rows_out);
/* Greedy evaluation sweep = evaluate() (proj/src/tuner.cpp:266-315):
 * inference over every shader, per-app aggregation with
 * run_seed = derive_seed({seed, 0x45564C, app}), uplift rows + histogram.
 * Host outputs: rows_out [n_apps][5] (as gbxcu_aggregate), histogram as
 * gbxcu_histogram (nullable). shader_actions_out [n_shaders] nullable. */
int gbxcu_evaluate(gbxcu_ctx* ctx, const gbxcu_dsuite* s, const float* params, int n_samples,
                   uint64_t seed, double* rows_out, uint8_t* shader_actions_out,
                   double* hist_lower, uint64_t* hist_count, size_t hist_cap, size_t* n_bins);
/* Device form: params, actions and rows are device buffers; no host sync. */
int gbxcu_evaluate_dev(gbxcu_ctx* ctx, const gbxcu_dsuite* s, const float* d_params,
                       int n_samples, uint64_t seed, uint8_t* d_actions, double* d_rows,
                       void* stream);

/* ------------------------------------------------ wide MLP variant (C4) */
/* 44 -> H -> H -> 2 policy (H multiple of 32, <= 1024) trained on the
 * tcgen05 tensor cores in TF32 with fp32 accumulation (BASELINE.json config
 * C4). Same algorithm as fit (shuffle, KL loss, analytic gradient, SGD),
 * generalised over widths; the reference hard-codes 44-64-32-2
 * (proj/include/gbx/policy.hpp:32-35), so parity is tolerance-based against
 * the generic oracle. Parameters use the same flat serialization order:
 * w0[H][44] b0[H] w1[H][H] b1[H] w2[2][H] b2[2]. */
size_t gbxcu_wide_param_count(int hidden);
int gbxcu_wide_init(gbxcu_ctx* ctx, int hidden, uint64_t seed, float* params_out);
int gbxcu_wide_forward(gbxcu_ctx* ctx, int hidden, const float* params, const float* feat, size_t n,
                       double* probs_out);
int gbxcu_wide_fit(gbxcu_ctx* ctx, int hidden, float* params_inout, const float* feat,
                   const double* tgt, size_t n, const gbxcu_train_cfg* cfg, double* epoch_loss_out,
                   int* diverged_epoch);
int gbxcu_wide_fit_dev(gbxcu_ctx* ctx, int hidden, float* d_params, const float* d_feat,
                       const double* d_tgt, size_t n, const gbxcu_train_cfg* cfg,
                       double* epoch_loss_out, int* diverged_epoch, void* stream);
/* Precision of the wide path: TF32 operands (kind::tf32, fp32 activations)
 * or BF16 operands (kind::f16; bf16 activations between the GEMMs, the
 * softmax/KL head fused into the layer-2 GEMM epilogue, fp32 master weights;
 * hidden a multiple of 64 up to 512). gbxcu_wide_fit[_dev] = TF32. */
#define GBXCU_WIDE_TF32 0
#define GBXCU_WIDE_BF16 1
int gbxcu_wide_fit_ex(gbxcu_ctx* ctx, int hidden, int precision, float* params_inout, const float* feat,
                      const double* tgt, size_t n, const gbxcu_train_cfg* cfg, double* epoch_loss_out,
                      int* diverged_epoch);
int gbxcu_wide_fit_ex_dev(gbxcu_ctx* ctx, int hidden, int precision, float* d_params, const float* d_feat,
                          const double* d_tgt, size_t n, const gbxcu_train_cfg* cfg, double* epoch_loss_out,
                          int* diverged_epoch, void* stream);
/* D[M][N] = A[M][K] . B[N][K]^T through the same tcgen05 TF32 GEMM kernel
 * (host buffers; K multiple of 4) — exposed for testing. */
int gbxcu_tf32_gemm(gbxcu_ctx* ctx, int M, int N, int K, const float* A, const float* B, float* D);
/* D[M][N] = bf16(A)[M][K] . bf16(B)[N][K]^T (round-to-nearest-even operands,
 * fp32 accumulation) through the wide path's kind::f16 kernel — for testing. */
int gbxcu_bf16_gemm(gbxcu_ctx* ctx, int M, int N, int K, const float* A, const float* B, float* D);

#ifdef __cplusplus
}
#endif
#endif /* GBXCU_H */
