// kernels.h — kernel declarations shared between the .cu translation units.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace gbxcu {

constexpr int FWD_BLOCK = 256;    // fast inference: 8 warps, two states per thread
constexpr int EXACT_BLOCK = 128;  // exact fp64 inference
constexpr int RECHECK_BLOCK = 256;  // warp-per-state exact re-check
constexpr int TRAIN_BLOCK = 512;  // train: 16 warps; tiles of 32 or 64 records
constexpr int SHUF_BLOCK = 256;
constexpr int AGG_BLOCK = 256;    // aggregation: 8 warps per CTA
constexpr int AGG_APPS = 4;       // aggregation: apps folded together by one warp (lane j = app j)
constexpr int AGG_MINB = 3;       // aggregation: resident CTAs per SM the register budget targets

constexpr int PSTR = 5028;        // per-CTA partial row: 5,026 gradient entries, loss, pad
constexpr int MAX_PEERS = 8;      // ranks of one NVLink domain (one node)
// Peer sets (k_train_tc.cu): per-GPU sums cross NVLink as LL word pairs
// {tag:32 | low 32 bits}, {tag:32 | high 32 bits}; the loss pair sits after
// the parameters.

// mode bits for the inference kernels
constexpr int FWD_PROBS = 1, FWD_ACTIONS = 2, FWD_COLLECT = 4, FWD_SAMPLE = 8;

struct TrainArgs {
    const float* feat;
    const double* tgt;
    const uint32_t* order;
    float* params;         // fp32 master copy (updated in place)
    double* partials;      // [gridDim][NP+1] per-CTA gradient + loss partials
    unsigned int* bar;     // grid-barrier counter (zeroed before launch)
    int* diverged_epoch;   // -1 until a non-finite batch loss
    double* epoch_loss;    // [epochs]
    size_t n;
    int batch;
    int epoch;
    double lr;
    int rank, nranks;
    // multi-CTA epoch kernel (k_train_tc.cu): data-flow step synchronisation
    // over a peer set — one process per GPU exchanging through NVLink peer
    // memory, or (pvirt) every rank inside one launch for single-GPU tests.
    int peers;                               // ranks in the set (1 = this GPU alone)
    int prank;                               // this process's rank in the set
    int pvirt;                               // 1: rank = blockIdx.x / (gridDim.x / peers)
    unsigned long long* ctr[MAX_PEERS];      // arrival counters (monotonic over fits)
    unsigned long long* llp[MAX_PEERS];      // {tag, fp32 bits} parameter words [NP]
    double* part[MAX_PEERS];                 // per-CTA partial rows [G][PSTR] (rank-local reads)
    unsigned long long* gp[MAX_PEERS];       // LL per-GPU sums: pairs [NP] params, [NP] loss
    unsigned int tag_base;                   // steps taken on this peer set before the epoch
    unsigned long long ctr_base;             // counter value before the epoch's first step
    // variants (0 = the reference's KL + SGD)
    int loss_mode;                           // 1: TD / reward regression of Q(x, a)
    int optimizer;                           // 1: Adam
    double beta1, beta2, adam_eps;
    double* adam_m;                          // [NP] first moments (slice-owned)
    double* adam_v;                          // [NP] second moments
    unsigned int step0;                      // optimizer steps taken before this epoch
    int* status;                             // watchdog: 1 = a peer wait timed out
};

struct AggArgs {
    size_t n_apps;
    const uint64_t* app_pipe_off;
    const uint64_t* pipe_slot_off;
    const uint32_t* slot_shader;
    const double* slot_frac;
    const double* pipe_wt;
    const double* shader_lat;
    const double* app_f64;
    const uint8_t* shader_action;
    const uint64_t* run_seed;  // nullable: derive from eval_seed
    uint64_t eval_seed;
    int n_samples;
    double* rows;              // [n_apps][5]
    double* samples;           // nullable [n_apps][n_samples]
    size_t app_base;           // global index of app 0 (seeds of an app-range shard)
};
__global__ void slot_shader_range_kernel(const uint32_t* slot_shader, uint64_t s_lo, uint64_t s_hi,
                                         unsigned int* range /* [min, max] */);

__global__ void policy_init_kernel(uint64_t seed, float* params);
__global__ void fwd_fast_kernel(const float* params, const float* feat, size_t n, double* probs,
                                uint8_t* actions, const uint64_t* seg_off, size_t nseg,
                                const uint64_t* seg_seed, double eps, uint32_t* recheck,
                                unsigned int* n_recheck, unsigned int* flags, int mode);
__global__ void fwd_exact_kernel(const float* params, const float* feat, size_t n,
                                 const uint32_t* list, const unsigned int* n_list, double* probs,
                                 uint8_t* actions, const uint64_t* seg_off, size_t nseg,
                                 const uint64_t* seg_seed, double eps, unsigned int* flags,
                                 int mode);
__global__ void fwd_recheck_kernel(const float* params, const float* feat, const uint32_t* list,
                                   const unsigned int* n_list, double* probs, uint8_t* actions,
                                   const uint64_t* seg_off, size_t nseg, const uint64_t* seg_seed,
                                   double eps, int mode);
size_t fast_smem_bytes();
size_t exact_smem_bytes();
size_t recheck_smem_bytes();

template <int TB>
__global__ void train_epoch_kernel(TrainArgs a);
// batch <= 32 on one rank: the same bit-exact step on a TRAIN_CLUSTER-CTA cluster (k_train_cl.cu)
constexpr int TRAIN_CLUSTER = 4;
__global__ void train_epoch_cluster_kernel(TrainArgs a);
size_t train_cl_smem_bytes();
template <int TB>
__global__ void train_partial_kernel(TrainArgs a, long step);
template <int MT, bool SYS, bool VAR>
__global__ void train_epoch_tc_kernel(TrainArgs a);
template <int MT>
__global__ void train_partial_tc_kernel(TrainArgs a, long step);
size_t train_tc_smem_bytes(int mt);
__global__ void reduce_partials_kernel(const double* partials, int nctas, double* red,
                                       const int* diverged);
__global__ void apply_update_kernel(float* params, const double* red, double lr, size_t nb,
                                    int epoch, int* diverged, double* epoch_acc);
__global__ void finish_epoch_kernel(const double* epoch_acc, size_t n, int epoch,
                                    const int* diverged, double* out);
__global__ void batch_grad_kernel(TrainArgs a, double* grad_out, double* loss_out);
size_t train_smem_bytes(int tb);

__global__ void iota_kernel(uint32_t* order, size_t n);
struct ShuffleArgs {
    const uint32_t* in;   // order before this epoch's pass
    uint32_t* out;        // order after it
    uint32_t n;
    uint64_t seed_e;      // derive_seed({seed, 0x5F17, epoch})
    uint32_t *jp, *head, *nxt, *succ, *root, *root2;  // [n] scratch each
    uint32_t* fg0;
    unsigned int* flags;  // [64] zeroed: "pointer jumping changed something in round r"
    unsigned int* bar;    // grid-barrier counter, zeroed
    const int* diverged;
};
__global__ void shuffle_epoch_kernel(ShuffleArgs s);

// ---------------------------------------------------------- wide MLP (C4)
enum GemmEpi { EPI_STORE = 0, EPI_BIAS_RELU = 1, EPI_MASK_T = 2 };

struct GemmArgs {
    int M, N, K;
    const float* A;          // [M][lda], K-major (rows optionally gathered)
    int lda;
    const uint32_t* a_rows;  // nullable row indirection for A
    const float* B;          // [N][ldb], K-major
    int ldb;
    int epi;
    const float* bias;       // EPI_BIAS_RELU
    float* out;              // row-major [M][ldo] (EPI_STORE: + blockIdx.z * split_stride)
    int ldo;
    float* out_t;            // transposed [N][ldt]
    int ldt;
    const float* mask;       // EPI_MASK_T: [M][ldm]
    int ldm;
    size_t split_stride;
};

struct WideHeadArgs {
    const float* h2;        // [nb][hidden]
    const float* w2;        // [2][hidden]
    const float* b2;        // [2]
    const double* tgt;      // targets, indexed through rows
    const uint32_t* rows;   // nullable
    int nb, hidden, ldt;
    double inv_b;
    double* kl;             // [nb]
    float* d3;              // [nb][2]
    float* d2;              // [nb][hidden]
    float* d2t;             // [hidden][ldt]
    double* part;           // [blocks][3*hidden + 3]: gW2 rows, gb1, gb2, KL sums of the block
};
__global__ void wide_head_reduce_kernel(const double* part, int nblocks, int hidden, float* gw2,
                                        float* gb2, float* gb1, double* loss_out);

// ---- wide MLP, BF16 tensor-core path (k_wide16.cu)
constexpr int W16_MAX_H = 512;   // the fused head: a CTA pair (2 x 256 TMEM columns) covers a full row
constexpr int W16_EPI_H1 = 0;    // relu(acc + bias) -> bf16 row-major + transposed
constexpr int W16_EPI_HEAD = 1;  // fused softmax/KL head over full rows
constexpr int W16_EPI_D1T = 2;   // acc [mask > 0] -> bf16 transposed
constexpr int W16_EPI_PART = 3;  // fp32 split-K partials
constexpr int W16_EPI_SGD = 4;   // gW1 and [gW0|gb0] tiles, split-K over W16_SPLITS-CTA clusters -> SGD
                                 // of every parameter + bf16 copies (one launch, no update kernel)
constexpr int W16_SPLITS = 6;    // K splits (= cluster size along z) of the fused SGD epilogues:
                                 // 22 clusters of 6 fit on 148 SMs at once (of 7 or 8: 15 < 16 tiles)
struct W16UpdArgs {
    float* params;                 // fp32 master weights (flat serialization order)
    int hidden;
    size_t np, nb;
    double lr;
    const float* p4;               // gW1 partials [s4][H][H]
    int s4;
    const float* p5;               // gW0|gb0 partials [s5][H][64]
    int s5;
    const double* hp;              // head partials [nhead][3H + 3]
    int nhead;
    float* g_out;                  // flat gradient (data-parallel path)
    double* loss_sum;              // KL sum (data-parallel path)
    __nv_bfloat16 *w0p, *w1, *w1t; // bf16 operand copies
    const int* epoch;
    int* diverged;
    double* epoch_acc;
    int dbg;                       // timeline slot (GBX_PHASE_TIMING builds), -1 = none
};
struct W16Args {
    int M, N, K;
    const float* bias;             // H1: b0, HEAD: b1
    __nv_bfloat16* out;            // row-major [M][ldo] (H1, D2)
    int ldo;
    __nv_bfloat16* out_t;          // transposed [N][ldt] (H1^T, D2^T, D1^T)
    int ldt;
    const __nv_bfloat16* mask;     // D1T: H1 [M][ldm]
    int ldm;
    float* part;                   // PART: [split][M][ldp]
    int ldp;
    size_t split_stride;
    // HEAD
    const float* w2;               // [2][N]
    const float* b2;               // [2]
    const double* tgt;             // targets, indexed through rows
    const uint32_t* rows;          // nullable
    double inv_b;
    double* head_part;             // [row tiles][3N + 3]: gW2_0, gW2_1, gb1, gb2_0, gb2_1, KL
    int dbg;                       // timeline slot (GBX_PHASE_TIMING builds), -1 = none
    W16UpdArgs u;                  // SGD1 / SGD0: the step's update
};
// epilogue warps per TMEM lane quarter of w16_gemm_kernel<.., EPI> (128 x this threads)
template <int EPI>
__host__ __device__ constexpr int w_ew() { return EPI == W16_EPI_HEAD ? 4 : 4; }
template <int BN, int ST>
size_t w16_gemm_smem_bytes();
template <int BN, int ST, int EPI>
__global__ void w16_gemm_kernel(const __grid_constant__ CUtensorMap map_a,
                                const __grid_constant__ CUtensorMap map_b,
                                const __grid_constant__ CUtensorMap map_o,
                                const __grid_constant__ CUtensorMap map_ot, W16Args g);
__global__ void w16_gather_kernel(const float* feat, const uint32_t* rows, int nb, int dbg, __nv_bfloat16* xg,
                                  __nv_bfloat16* xt, int ldt);
__global__ void w16_weights_kernel(const float* params, int H, __nv_bfloat16* w0p, __nv_bfloat16* w1,
                                   __nv_bfloat16* w1t);
__global__ void w16_update_kernel(W16UpdArgs u, int mode);
__host__ __device__ void w16_update_layout(int H, size_t np, int& nb0, int& nw1, int& nb2);
__global__ void to_bf16_kernel(const float* src, size_t n, __nv_bfloat16* dst);

__global__ void tc_gemm_kernel(GemmArgs g);
template <int BN>
size_t tma_gemm_smem_bytes();
size_t gemm_smem_bytes();
__global__ void wide_gather_xt_kernel(const float* feat, const uint32_t* rows, int nb, float* xt,
                                      int ldt, float* xg);
__global__ void wide_head_kernel(WideHeadArgs a);
__global__ void row_sum_kernel(const float* in, int ld, int ncols, float* out);
__global__ void wide_w2_partial_kernel(const float* h2, const float* d3, const double* kl, int nb,
                                       int hidden, double* part);
__global__ void split_reduce_f32_kernel(const float* src, int splits, size_t stride, int rows,
                                        int cols, int ld_src, float* dst, int ld_dst);
__global__ void split_reduce_f64_kernel(const double* src, int splits, int n, float* dst,
                                        double* loss_out);
__global__ void wide_update_kernel(float* params, const float* grad, const double* loss_sum,
                                   size_t nb, double lr, int hidden, float* w1t, float* w0p,
                                   const int* epoch, int* diverged, double* epoch_acc, size_t np);
__global__ void wide_w1t_kernel(const float* params, int hidden, float* w1t, float* w0p);
__global__ void wide_gw0_kernel(const float* src, int splits, size_t stride, int hidden, float* dst,
                                float* gb0);
__global__ void wide_init_kernel(uint64_t seed, int hidden, float* params, size_t np);
__global__ void wide_probs_kernel(const float* h2, const float* w2, const float* b2, int nb,
                                  int hidden, double* probs);
__global__ void zero_cols_kernel(float* m, int rows, int ld, int c_lo, int c_hi);

// ------------------------------------------------- Q-table (row f1)
constexpr int QT_KEY_WORDS = 30;  // StateKey: stage + 29 raw counters
struct RecView;
struct FoldArgs;
__global__ void qt_iota_kernel(uint32_t* p, size_t n);
__global__ void qt_init_ids_kernel(const uint8_t* has, size_t m, uint32_t* ids, unsigned long long* count);
__global__ void qt_both_kernel(const uint8_t* has, size_t m, uint32_t* flag);
__global__ void qt_rowkey_kernel(const uint32_t* flag, const uint32_t* row, size_t m, uint32_t* rowkey);
constexpr uint32_t QT_ENC_TAB = 1u << 16;  // log1pf(count) table: counts below this
__global__ void qt_enc_table_kernel(float* tab);
__global__ void qt_snapshot_kernel(const uint32_t* keys, const double* q, const uint32_t* rowkey,
                                   size_t nrows, double rho, const float* enc_tab, float* feat, double* tgt,
                                   int* bad_stage);
// fold pipeline entry points (launch wrappers live in k_qtable.cu)
struct QtFoldIO {
    const uint32_t* tkeys; const uint32_t* init; size_t n_init;
    const uint32_t* bkeys; const uint8_t* bact; const double* reward; const uint64_t* now; size_t n;
    size_t limit;
    const double* old_q; const uint64_t* old_t; const uint64_t* old_cnt;
    double alpha, omega;
    // scratch [nrec] each
    uint32_t *perm, *perm2, *digit, *digit2, *seg_head, *key_head, *seg_scan, *key_scan, *seg_start, *seg_key;
    uint32_t* spread;            // [64]: sample spread, unresolved flag, exact spread
    void* rn;                    // [n] 16-byte (reward bits, check-in) per tuple
    void* temp; size_t temp_bytes;
    unsigned long long* bad;     // [1]
};
size_t qt_temp_bytes(size_t nrec);
// Sorts and segments the records; returns segment and key counts (synchronous).
cudaError_t qt_sort_segment(QtFoldIO& io, size_t& nseg, size_t& nkeys, int num_sms, cudaStream_t st);
// Folds into a new table (keys, q, t, cnt, has zeroed by the caller).
cudaError_t qt_fold(const QtFoldIO& io, size_t nseg, size_t nkeys, uint32_t* keys, double* q, uint64_t* t,
                    uint64_t* cnt, uint8_t* has, int num_sms, cudaStream_t st);
cudaError_t qt_exclusive_scan(void* temp, size_t temp_bytes, const uint32_t* in, uint32_t* out,
                              size_t n, cudaStream_t st);

template <int K, int MINB>
__global__ void aggregate_kernel(AggArgs a);
__global__ void histogram_kernel(const double* rows, int stride, size_t n, double* lower,
                                 unsigned long long* count, size_t cap,
                                 unsigned long long* n_bins);

}  // namespace gbxcu
