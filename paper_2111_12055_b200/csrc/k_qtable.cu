// k_qtable.cu — the experience store on the device:
// QTable::update folded over a batch of tuples, and snapshot_policy_dataset
// producing fit's training records in key order.
//
// Reference: QTable::update (proj/src/qtable.cpp:76-92), boltzmann_pair
// (:121-129), snapshot_policy_dataset (:143-155) -> counters_from_key +
// encode_state (proj/src/core.cpp:43-62,105-123), RawCounters::recompute_totals
// (proj/src/core.cpp:19-28); StateKey order = lexicographic over 30 u32
// (proj/include/gbx/core.hpp:126-130).
//
// Fold of n tuples (key, action, reward, check-in) into a table of m states:
//   1. records = the table's existing entries (as "init" records, first) +
//      the tuples in sequence order;
//   2. stable LSD radix sort of the record permutation by (key words 0..29,
//      action): action first, then word 29 .. word 0; words whose values are
//      all equal are skipped, the others contribute only their varying low
//      bits, packed into 64-bit digits (one gather + one cub::DeviceRadixSort
//      per 64 bits; the sorts are the only library calls);
//   3. segment heads by comparing neighbours (key, action) and key alone;
//   4. one thread per (key, action) segment folds its records in sequence
//      order — the Eq.-5 recurrence is a strict left fold, so each segment is
//      sequential, exactly like the reference; different segments in parallel:
//          q <- ((1 - alpha) * omega^dt) * q + alpha * r   (no FMA, as g++)
//      A check-in earlier than the entry's timestamp is a ClockRegressionError:
//      the smallest such tuple index is reported, and the host re-folds the
//      prefix before it so the table ends exactly where the reference's does;
//   5. the new table (unique keys in order, per-action entries) replaces the old.
// Snapshot: keys with both actions, compacted in key order; features =
// encode_state(counters_from_key(key)) with glibc's log1pf restated bit for bit
// (fdlibm algorithm, no FMA contraction), targets = boltzmann_pair(q0, q1, rho).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "common.cuh"
#include "kernels.h"

namespace gbxcu {

constexpr int KW = QT_KEY_WORDS;  // 30

// ---------------------------------------------------------------- records
// Key words of record i: existing entries come from the table, tuples from
// the batch. rec < n_init: table entry rec (key row rec >> 1, action rec & 1).
struct RecView {
    const uint32_t* tkeys;   // [m][30] table keys
    const uint32_t* init;    // [n_init] table entry ids (key * 2 + action)
    size_t n_init;
    const uint32_t* bkeys;   // [n][30] batch keys
    const uint8_t* bact;     // [n]
    __device__ __forceinline__ const uint32_t* key(uint32_t rec) const {
        return rec < n_init ? tkeys + (size_t)(init[rec] >> 1) * KW : bkeys + (size_t)(rec - n_init) * KW;
    }
    __device__ __forceinline__ uint32_t action(uint32_t rec) const {
        return rec < n_init ? (init[rec] & 1u) : (uint32_t)bact[rec - n_init];
    }
};

__global__ void qt_iota_kernel(uint32_t* p, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        p[i] = (uint32_t)i;
}

// Existing entries of the table as init records: ids key*2 + action of present entries.
__global__ void qt_init_ids_kernel(const uint8_t* __restrict__ has, size_t m, uint32_t* __restrict__ ids,
                                   unsigned long long* __restrict__ count) {
    for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < m; k += (size_t)gridDim.x * blockDim.x) {
        for (int a = 0; a < 2; ++a)
            if (has[2 * k + a]) ids[atomicAdd(count, 1ull)] = (uint32_t)(2 * k + a);
    }
}

// Per key word: OR of (v ^ word of record 0) (which bits vary) over the
// records 0, stride, 2 stride, ... (stride 1: all records).
__global__ void qt_word_spread_kernel(RecView v, size_t nrec, size_t stride, uint32_t* __restrict__ spread) {
    __shared__ uint32_t acc[KW + 1];
    if (threadIdx.x <= KW) acc[threadIdx.x] = 0;
    __syncthreads();
    const uint32_t* k0 = v.key(0);
    const uint32_t a0 = v.action(0);
    uint32_t loc[KW + 1];
#pragma unroll
    for (int w = 0; w <= KW; ++w) loc[w] = 0;
    const size_t ns = (nrec + stride - 1) / stride;
    for (size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x; j < ns; j += (size_t)gridDim.x * blockDim.x) {
        const uint32_t i = (uint32_t)(j * stride);
        const uint32_t* k = v.key(i);
#pragma unroll
        for (int w = 0; w < KW; ++w) loc[w] |= k[w] ^ k0[w];
        loc[KW] |= v.action(i) ^ a0;
    }
#pragma unroll
    for (int w = 0; w <= KW; ++w) {
        uint32_t x = loc[w];
        for (int o = 16; o > 0; o >>= 1) x |= __shfl_xor_sync(0xffffffffu, x, o);
        if ((threadIdx.x & 31) == 0 && x) atomicOr(&acc[w], x);
    }
    __syncthreads();
    if (threadIdx.x <= KW && acc[threadIdx.x]) atomicOr(&spread[threadIdx.x], acc[threadIdx.x]);
}

// The fold's one sequential pass over the records (in record order): the MSD
// digit under a packing chosen from a sample of the records (per word: mask
// of its field, bit offset; index KW = the action), the exact word spread
// (checked by the host against that packing — a bit the sample missed means
// a re-run with the exact one), and the tuples' (reward, check-in) packed
// into one 16-byte record so the fold's per-record gather is one load.
struct WordPack {
    uint32_t mask[KW + 1];
    uint32_t off[KW + 1];
};
template <bool V2>
__global__ void __launch_bounds__(256) qt_first_pass_kernel(RecView v, size_t nrec, WordPack wp,
                                                            unsigned long long* __restrict__ digit,
                                                            uint32_t* __restrict__ spread,
                                                            const double* __restrict__ reward,
                                                            const uint64_t* __restrict__ now,
                                                            ulonglong2* __restrict__ rn) {
    __shared__ uint32_t acc[KW + 1];
    if (threadIdx.x <= KW) acc[threadIdx.x] = 0;
    __syncthreads();
    uint32_t k0[KW], loc[KW + 1];
    {
        const uint32_t* r0 = v.key(0);
#pragma unroll
        for (int w = 0; w < KW; ++w) k0[w] = __ldg(r0 + w);
    }
    const uint32_t a0 = v.action(0);
#pragma unroll
    for (int w = 0; w <= KW; ++w) loc[w] = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nrec; i += (size_t)gridDim.x * blockDim.x) {
        const uint32_t* k = v.key((uint32_t)i);
        uint32_t x[KW];
        if (V2) {  // rows are 120 bytes: 8-byte aligned when the base is
            const uint2* k2 = reinterpret_cast<const uint2*>(k);
#pragma unroll
            for (int q = 0; q < KW / 2; ++q) {
                const uint2 t = __ldg(k2 + q);
                x[2 * q] = t.x;
                x[2 * q + 1] = t.y;
            }
        } else {
#pragma unroll
            for (int w = 0; w < KW; ++w) x[w] = __ldg(k + w);
        }
        const uint32_t a = v.action((uint32_t)i);
        unsigned long long d = (unsigned long long)(a & wp.mask[KW]) << wp.off[KW];
#pragma unroll
        for (int w = 0; w < KW; ++w) {
            loc[w] |= x[w] ^ k0[w];
            d |= (unsigned long long)(x[w] & wp.mask[w]) << wp.off[w];
        }
        loc[KW] |= a ^ a0;
        digit[i] = d;
        if (i >= v.n_init) {
            const size_t b = i - v.n_init;
            rn[b] = make_ulonglong2((unsigned long long)__double_as_longlong(reward[b]), now[b]);
        }
    }
#pragma unroll
    for (int w = 0; w <= KW; ++w) {
        uint32_t x = loc[w];
        for (int o = 16; o > 0; o >>= 1) x |= __shfl_xor_sync(0xffffffffu, x, o);
        if ((threadIdx.x & 31) == 0 && x) atomicOr(&acc[w], x);
    }
    __syncthreads();
    if (threadIdx.x <= KW && acc[threadIdx.x]) atomicOr(&spread[threadIdx.x], acc[threadIdx.x]);
}

// One radix pass sorts a 64-bit digit packing several key words (only their
// varying low bits): field f = word wlist[f] (KW: the action), masked to
// bits[f], at bit offset off[f] (least significant field first).
struct PackSpec {
    int nf;
    int w[8];
    int bits[8];
    int off[8];
};
__global__ void qt_gather_digit_kernel(RecView v, const uint32_t* __restrict__ perm, size_t nrec, PackSpec ps,
                                       unsigned long long* __restrict__ digit) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nrec; i += (size_t)gridDim.x * blockDim.x) {
        const uint32_t r = perm[i];
        const uint32_t* k = v.key(r);
        unsigned long long d = 0;
        for (int f = 0; f < ps.nf; ++f) {
            const uint32_t x = ps.w[f] == KW ? v.action(r) : k[ps.w[f]];
            const uint32_t m = ps.bits[f] >= 32 ? 0xFFFFFFFFu : ((1u << ps.bits[f]) - 1u);
            d |= (unsigned long long)(x & m) << ps.off[f];
        }
        digit[i] = d;
    }
}

// Words [w_from, KW) of two keys equal? Both 120-byte rows are read with all
// fifteen 8-byte loads in flight at once (an early-exit word loop issues one
// dependent round trip per word).
__device__ __forceinline__ bool key_tail_equal(const uint32_t* a, const uint32_t* b, int w_from) {
    const uint2* a2 = reinterpret_cast<const uint2*>(a);
    const uint2* b2 = reinterpret_cast<const uint2*>(b);
    uint2 x[KW / 2], y[KW / 2];
#pragma unroll
    for (int q = 0; q < KW / 2; ++q) {
        x[q] = __ldg(a2 + q);
        y[q] = __ldg(b2 + q);
    }
    bool same = true;
#pragma unroll
    for (int q = 0; q < KW / 2; ++q) {
        if (2 * q >= w_from) same &= x[q].x == y[q].x;
        if (2 * q + 1 >= w_from) same &= x[q].y == y[q].y;
    }
    return same;
}
static_assert(KW % 2 == 0, "keys are read as 8-byte pairs");

// MSD fast path: segment heads straight from the sorted digits (key bits
// above `abits` action bits), plus the check that makes them valid —
// neighbours with equal key bits must have equal keys (words w_from.. beyond
// the digit; none when w_from == KW), else the order is unresolved and the
// caller falls back to the full LSD sort. With abits == 0 every record has
// the same action. Warp-wide over 32 consecutive positions: a row needed by
// a tie is loaded once, by its own lane, and handed to the next lane by
// shuffles (lane 0 loads its predecessor itself).
__global__ void qt_msd_heads_kernel(RecView v, const uint32_t* __restrict__ perm,
                                    const unsigned long long* __restrict__ digit, size_t nrec,
                                    int w_from, int abits, unsigned int* __restrict__ unresolved,
                                    uint32_t* __restrict__ seg_head, uint32_t* __restrict__ key_head) {
    const int lane = threadIdx.x & 31;
    const size_t step = (size_t)gridDim.x * blockDim.x;
    for (size_t base = blockIdx.x * (size_t)blockDim.x + threadIdx.x - lane; base < nrec; base += step) {
        const size_t i = base + lane;
        const bool act = i < nrec;
        const unsigned long long d = act ? digit[i] : 0ull;
        const unsigned long long dp = (act && i > 0) ? digit[i - 1] : 0ull;
        const bool tie = act && i > 0 && (d >> abits) == (dp >> abits);
        uint32_t kh = tie ? 0u : 1u;
        if (w_from < KW && __any_sync(0xffffffffu, tie)) {
            bool tie_next = __shfl_down_sync(0xffffffffu, tie, 1);
            if (lane == 31) tie_next = i + 1 < nrec && (digit[i + 1] >> abits) == (d >> abits);
            const uint2* own = act ? reinterpret_cast<const uint2*>(v.key(perm[i])) : nullptr;
            const bool need = tie || tie_next;
            bool same = true;
            if (lane == 0 && tie) same = key_tail_equal(v.key(perm[i]), v.key(perm[i - 1]), w_from);
            uint2 xs[KW / 2];  // all loads in flight before the first shuffle
#pragma unroll
            for (int q = 0; q < KW / 2; ++q)
                xs[q] = need && 2 * q + 1 >= w_from ? __ldg(own + q) : make_uint2(0u, 0u);
#pragma unroll
            for (int q = 0; q < KW / 2; ++q) {
                const uint2 x = xs[q];
                const uint32_t yx = __shfl_up_sync(0xffffffffu, x.x, 1);
                const uint32_t yy = __shfl_up_sync(0xffffffffu, x.y, 1);
                if (lane > 0) {
                    if (2 * q >= w_from) same &= x.x == yx;
                    if (2 * q + 1 >= w_from) same &= x.y == yy;
                }
            }
            if (tie && !same) {
                atomicOr(unresolved, 1u);
                kh = 1;
            }
        }
        if (act) {
            seg_head[i] = kh | (uint32_t)((d ^ dp) & (unsigned long long)abits);
            key_head[i] = kh;
        }
    }
}

// seg_head[i]: (key, action) differs from position i-1; key_head[i]: key differs.
__global__ void qt_heads_kernel(RecView v, const uint32_t* __restrict__ perm, size_t nrec,
                                uint32_t* __restrict__ seg_head, uint32_t* __restrict__ key_head) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nrec; i += (size_t)gridDim.x * blockDim.x) {
        uint32_t kh = 1, sh = 1;
        if (i > 0) {
            kh = key_tail_equal(v.key(perm[i]), v.key(perm[i - 1]), 0) ? 0u : 1u;
            sh = kh | (v.action(perm[i]) != v.action(perm[i - 1]) ? 1u : 0u);
        }
        seg_head[i] = sh;
        key_head[i] = kh;
    }
}

// Segment starts (positions with seg_head) and, per segment, its key index.
__global__ void qt_seg_list_kernel(const uint32_t* __restrict__ seg_head, const uint32_t* __restrict__ seg_scan,
                                   const uint32_t* __restrict__ key_scan, size_t nrec,
                                   uint32_t* __restrict__ seg_start, uint32_t* __restrict__ seg_key) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nrec; i += (size_t)gridDim.x * blockDim.x) {
        if (seg_head[i]) {
            const uint32_t s = seg_scan[i];  // exclusive scan: segment id
            seg_start[s] = (uint32_t)i;
            seg_key[s] = key_scan[i] - 1;    // inclusive scan of key heads - 1
        }
    }
}

struct FoldArgs {
    RecView v;
    const uint32_t* perm;
    size_t nrec, nseg;
    const uint32_t* seg_start;
    const uint32_t* seg_key;
    // old table entries (init records)
    const double* old_q;
    const uint64_t* old_t;
    const uint64_t* old_cnt;
    // batch: (reward bits, check-in) per tuple, packed by the first pass
    const ulonglong2* rn;
    size_t limit;            // tuples with batch index >= limit are ignored (prefix re-fold)
    double alpha, omega;
    // new table
    uint32_t* keys;          // [m'][30]
    double* q;               // [m'][2]
    uint64_t* t;
    uint64_t* cnt;
    uint8_t* has;
    unsigned long long* bad; // min batch index of a ClockRegressionError
    uint32_t* src_rec;       // [m'] a record carrying each written key (0xFFFFFFFF: none)
};

// One thread per (key, action) segment: QTable::update in sequence order.
__global__ void qt_fold_kernel(FoldArgs f) {
    for (size_t s = blockIdx.x * (size_t)blockDim.x + threadIdx.x; s < f.nseg; s += (size_t)gridDim.x * blockDim.x) {
        const size_t lo = f.seg_start[s];
        const size_t hi = s + 1 < f.nseg ? f.seg_start[s + 1] : f.nrec;
        const uint32_t kid = f.seg_key[s];
        const uint32_t first = f.perm[lo];
        const int a = (int)f.v.action(first);
        bool have = false;
        double q = 0.0;
        uint64_t t = 0, cnt = 0;
        for (size_t i = lo; i < hi; ++i) {
            const uint32_t r = f.perm[i];
            if (r < f.v.n_init) {  // existing entry (always first in its segment)
                const uint32_t e = f.v.init[r];
                q = f.old_q[e];
                t = f.old_t[e];
                cnt = f.old_cnt[e];
                have = true;
                continue;
            }
            const size_t b = r - f.v.n_init;
            if (b >= f.limit) break;  // batch order == record order within a segment
            const ulonglong2 p = f.rn[b];
            const double rw = __longlong_as_double((long long)p.x);
            const uint64_t now = p.y;
            if (!have) {  // slot = QEntry{r, now, 1}
                q = rw;
                t = now;
                cnt = 1;
                have = true;
                continue;
            }
            if (now < t) {  // ClockRegressionError: stop this segment, report the index
                atomicMin(f.bad, (unsigned long long)b);
                break;
            }
            const double dt = (double)(now - t);
            // (1.0 - alpha) * pow(omega, dt) * q + alpha * r, evaluated left to right
            const double decay = f.omega == 1.0 ? 1.0 : pow(f.omega, dt);
            q = __dadd_rn(__dmul_rn(__dmul_rn(__dsub_rn(1.0, f.alpha), decay), q), __dmul_rn(f.alpha, rw));
            t = now;
            cnt += 1;
        }
        if (!have) continue;  // only tuples past `limit`
        const size_t e = 2 * (size_t)kid + a;
        f.q[e] = q;
        f.t[e] = t;
        f.cnt[e] = cnt;
        f.has[e] = 1;
        // the key row is copied by qt_copy_keys_kernel (coalesced); either
        // segment of the key names a record with the same words
        f.src_rec[kid] = first;
    }
}

// New key rows: thread per (key, word), so a warp reads and writes whole
// 120-byte rows (a thread-per-key copy touches 30 sectors per instruction);
// four independent items per thread per iteration keep enough random row
// reads in flight.
__global__ void qt_copy_keys_kernel(RecView v, const uint32_t* __restrict__ src_rec, size_t nkeys,
                                    uint32_t* __restrict__ keys) {
    constexpr int U = 4;
    const size_t total = nkeys * KW;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t x0 = blockIdx.x * (size_t)blockDim.x + threadIdx.x; x0 < total; x0 += U * stride) {
        uint32_t r[U], val[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t x = x0 + u * stride;
            r[u] = x < total ? __ldg(src_rec + x / KW) : 0xFFFFFFFFu;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t x = x0 + u * stride;
            if (r[u] != 0xFFFFFFFFu) val[u] = __ldg(v.key(r[u]) + (x - (x / KW) * KW));
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (r[u] != 0xFFFFFFFFu) keys[x0 + u * stride] = val[u];
    }
}

// ------------------------------------------------------------- snapshot
// glibc 2.39 log1pf (sysdeps/ieee754/flt-32/s_log1pf.c, fdlibm), restated with
// explicit fp32 rounding so nvcc cannot contract; bit-identical to the host's
// on every integer count (tools check: 0 mismatches over 1e8 values).
__device__ float glibc_log1pf(float x) {
    const float ln2_hi = 6.9313812256e-01f, ln2_lo = 9.0580006145e-06f;
    const float Lp1 = 6.6666668653e-01f, Lp2 = 4.0000000596e-01f, Lp3 = 2.8571429849e-01f,
                Lp4 = 2.2222198546e-01f, Lp5 = 1.8183572590e-01f, Lp6 = 1.5313838422e-01f,
                Lp7 = 1.4798198640e-01f;
    // counts are >= 0: only the x >= 0 branches of the reference are reachable
    int32_t hx = __float_as_int(x);
    if (hx == 0) return 0.0f;
    if (hx >= 0x7f800000) return __fadd_rn(x, x);
    int32_t k = 1, hu;
    float f, c, u;
    if (hx < 0x3ed413d7) {  // 0 < x < 0.41422: k = 0 (integers never land here except 0)
        k = 0;
        f = x;
        hu = 1;
        c = 0.0f;
    } else {
        if (hx < 0x5a000000) {
            u = __fadd_rn(1.0f, x);
            hu = __float_as_int(u);
            k = (hu >> 23) - 127;
            c = (k > 0) ? __fsub_rn(1.0f, __fsub_rn(u, x)) : __fsub_rn(x, __fsub_rn(u, 1.0f));
            c = __fdiv_rn(c, u);
        } else {
            u = x;
            hu = __float_as_int(u);
            k = (hu >> 23) - 127;
            c = 0.0f;
        }
        hu &= 0x007fffff;
        if (hu < 0x3504f7) {
            u = __int_as_float(hu | 0x3f800000);
        } else {
            k += 1;
            u = __int_as_float(hu | 0x3f000000);
            hu = (0x00800000 - hu) >> 2;
        }
        f = __fsub_rn(u, 1.0f);
    }
    const float hfsq = __fmul_rn(__fmul_rn(0.5f, f), f);
    const float fk = (float)k;
    if (hu == 0) {
        if (f == 0.0f) {
            if (k == 0) return 0.0f;
            c = __fadd_rn(c, __fmul_rn(fk, ln2_lo));
            return __fadd_rn(__fmul_rn(fk, ln2_hi), c);
        }
        const float R = __fmul_rn(hfsq, __fsub_rn(1.0f, __fmul_rn(0.66666666666666666f, f)));
        if (k == 0) return __fsub_rn(f, R);
        return __fsub_rn(__fmul_rn(fk, ln2_hi),
                         __fsub_rn(__fsub_rn(R, __fadd_rn(__fmul_rn(fk, ln2_lo), c)), f));
    }
    const float s = __fdiv_rn(f, __fadd_rn(2.0f, f));
    const float z = __fmul_rn(s, s);
    float R = __fadd_rn(Lp6, __fmul_rn(z, Lp7));
    R = __fadd_rn(Lp5, __fmul_rn(z, R));
    R = __fadd_rn(Lp4, __fmul_rn(z, R));
    R = __fadd_rn(Lp3, __fmul_rn(z, R));
    R = __fadd_rn(Lp2, __fmul_rn(z, R));
    R = __fadd_rn(Lp1, __fmul_rn(z, R));
    R = __fmul_rn(z, R);
    if (k == 0) return __fsub_rn(f, __fsub_rn(hfsq, __fmul_rn(s, __fadd_rn(hfsq, R))));
    return __fsub_rn(__fmul_rn(fk, ln2_hi),
                     __fsub_rn(__fsub_rn(hfsq, __fadd_rn(__fmul_rn(s, __fadd_rn(hfsq, R)),
                                                         __fadd_rn(__fmul_rn(fk, ln2_lo), c))),
                               f));
}

__device__ __forceinline__ float enc_count(uint32_t c) { return glibc_log1pf(__uint2float_rn(c)); }

// enc_count of every count below QT_ENC_TAB, computed by the same function
// (so a lookup is bit-identical): the snapshot encodes 36 counts per row and
// real counts are mostly small, so most of its ~150-instruction log1pf calls
// become one L1/L2-resident load.
__global__ void qt_enc_table_kernel(float* __restrict__ tab) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c < QT_ENC_TAB) tab[c] = enc_count(c);
}

// Row flags: key with both actions recorded.
__global__ void qt_both_kernel(const uint8_t* __restrict__ has, size_t m, uint32_t* __restrict__ flag) {
    for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < m; k += (size_t)gridDim.x * blockDim.x)
        flag[k] = (has[2 * k] && has[2 * k + 1]) ? 1u : 0u;
}

// One thread per key: encode_state(counters_from_key(key)) + boltzmann_pair.
// Row -> key map of the snapshot (rows = keys with both actions, key order).
__global__ void qt_rowkey_kernel(const uint32_t* __restrict__ flag, const uint32_t* __restrict__ row,
                                 size_t m, uint32_t* __restrict__ rowkey) {
    for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < m; k += (size_t)gridDim.x * blockDim.x)
        if (flag[k]) rowkey[row[k]] = (uint32_t)k;
}

// One warp per 32 consecutive output rows: the key rows are read
// cooperatively into shared memory (whole 120-byte rows per instruction),
// each lane encodes its row, and the 32 x 44 feature block is written back
// as one contiguous, coalesced range.
constexpr int SNAP_WARPS = 4;
__global__ void __launch_bounds__(SNAP_WARPS * 32, 5)
qt_snapshot_kernel(const uint32_t* __restrict__ keys, const double* __restrict__ q,
                   const uint32_t* __restrict__ rowkey, size_t nrows, double rho,
                   const float* __restrict__ enc_tab, float* __restrict__ feat, double* __restrict__ tgt,
                   int* __restrict__ bad_stage) {
    __shared__ uint32_t kt[SNAP_WARPS][32 * (KW + 1)];
    __shared__ float ft[SNAP_WARPS][32 * (F + 1)];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t* K = kt[w];
    float* Fo = ft[w];
    for (size_t r0 = ((size_t)blockIdx.x * SNAP_WARPS + w) * 32; r0 < nrows;
         r0 += (size_t)gridDim.x * SNAP_WARPS * 32) {
        const int nv = (int)min((size_t)32, nrows - r0);
        const uint32_t kl = lane < nv ? rowkey[r0 + lane] : 0u;
        // all 30 loads of the warp's rows in flight before the first store
        uint32_t kv[KW];
#pragma unroll
        for (int j = 0; j < KW; ++j) {
            const int x = 32 * j + lane, rr = x / KW, wd = x - rr * KW;
            const uint32_t kk = __shfl_sync(0xffffffffu, kl, rr & 31);
            kv[j] = rr < nv ? __ldg(keys + (size_t)kk * KW + wd) : 0u;
        }
#pragma unroll
        for (int j = 0; j < KW; ++j) {
            const int x = 32 * j + lane, rr = x / KW, wd = x - rr * KW;
            K[rr * (KW + 1) + wd] = kv[j];
        }
        __syncwarp();
        if (lane < nv) {
            const uint32_t* v = K + lane * (KW + 1);
            float* out = Fo + lane * (F + 1);
            const uint32_t stage = v[0];
            if (stage >= 8) {  // counters_from_key: "state key holds invalid stage index"
                atomicExch(bad_stage, 1);
            } else {
#pragma unroll
                for (int i = 0; i < 8; ++i) out[i] = i == (int)stage ? 1.0f : 0.0f;
                // slots 8..36: basic blocks, vector[5], scalar[4], memory[6], compute[4],
                // control-flow[4], registers[2], work groups[3] = key words 1..29
                // table loads issued together (clamped); counts past the table
                // are recomputed below
#pragma unroll
                for (int wd = 1; wd < KW; ++wd) out[7 + wd] = __ldg(enc_tab + min(v[wd], QT_ENC_TAB - 1));
#pragma unroll 1
                for (int wd = 1; wd < KW; ++wd)
                    if (v[wd] >= QT_ENC_TAB) out[7 + wd] = enc_count(v[wd]);
                // totals (u32 wrap, like the u64 sums cast back): vector, scalar, memory,
                // compute, control-flow, registers; instructions = the first five
                const int lo_[6] = {2, 7, 11, 17, 21, 25};
                const int len_[6] = {5, 4, 6, 4, 4, 2};
                uint32_t tot[7];
                for (int g = 0; g < 6; ++g) {
                    uint32_t sacc = 0;
                    for (int i = 0; i < len_[g]; ++i) sacc += v[lo_[g] + i];
                    tot[g + 1] = sacc;
                }
                tot[0] = tot[1] + tot[2] + tot[3] + tot[4] + tot[5];
#pragma unroll
                for (int i = 0; i < 7; ++i) out[37 + i] = __ldg(enc_tab + min(tot[i], QT_ENC_TAB - 1));
#pragma unroll
                for (int i = 0; i < 7; ++i)
                    if (tot[i] >= QT_ENC_TAB) out[37 + i] = enc_count(tot[i]);
            }
            // boltzmann_pair (qtable.cpp:121-129)
            const double q0 = q[2 * (size_t)kl], q1 = q[2 * (size_t)kl + 1];
            const double mx = q0 < q1 ? q1 : q0;  // std::max
            const double e0 = exp(__ddiv_rn(__dsub_rn(q0, mx), rho));
            const double e1 = exp(__ddiv_rn(__dsub_rn(q1, mx), rho));
            const double sm = __dadd_rn(e0, e1);
            tgt[2 * (r0 + lane)] = __ddiv_rn(e0, sm);
            tgt[2 * (r0 + lane) + 1] = __ddiv_rn(e1, sm);
        }
        __syncwarp();
        float* dst = feat + r0 * F;
        for (int x = lane; x < nv * F; x += 32) {
            const int rr = x / F;
            dst[x] = Fo[rr * (F + 1) + (x - rr * F)];
        }
        __syncwarp();
    }
}

// ------------------------------------------------------------ host helpers
size_t qt_temp_bytes(size_t n) {
    size_t a = 0, b = 0, c = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, a, (const unsigned long long*)nullptr,
                                    (unsigned long long*)nullptr, (const uint32_t*)nullptr,
                                    (uint32_t*)nullptr, (int)n);
    cub::DeviceScan::ExclusiveSum(nullptr, b, (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)n);
    cub::DeviceScan::InclusiveSum(nullptr, c, (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)n);
    return a > b ? (a > c ? a : c) : (b > c ? b : c);
}

cudaError_t qt_exclusive_scan(void* temp, size_t temp_bytes, const uint32_t* in, uint32_t* out, size_t n,
                              cudaStream_t st) {
    return cub::DeviceScan::ExclusiveSum(temp, temp_bytes, in, out, (int)n, st);
}

#define QT_CK(x)                                \
    do {                                        \
        cudaError_t e_ = (x);                   \
        if (e_ != cudaSuccess) return e_;       \
    } while (0)

static RecView rec_view(const QtFoldIO& io) {
    return RecView{io.tkeys, io.init, io.n_init, io.bkeys, io.bact};
}

cudaError_t qt_sort_segment(QtFoldIO& io, size_t& nseg, size_t& nkeys, int num_sms, cudaStream_t st) {
    const size_t nrec = io.n_init + io.n;
    const RecView v = rec_view(io);
    const int grid = num_sms * 4;
    qt_iota_kernel<<<grid, 256, 0, st>>>(io.perm, nrec);
    // spread[0..KW]: a sample's word spread; [KW + 1]: the unresolved flag;
    // [KW + 2 .. 2 KW + 2]: the exact spread from the first pass
    uint32_t* exact = io.spread + KW + 2;
    QT_CK(cudaMemsetAsync(io.spread, 0, sizeof(uint32_t) * (2 * KW + 3), st));
    const size_t stride = std::max<size_t>(1, nrec / 65536);
    qt_word_spread_kernel<<<grid, 256, 0, st>>>(v, nrec, stride, io.spread);
    uint32_t spread[KW + 1];
    QT_CK(cudaMemcpyAsync(spread, io.spread, sizeof(spread), cudaMemcpyDeviceToHost, st));
    QT_CK(cudaStreamSynchronize(st));
    auto bits_of = [&](int w) { return spread[w] ? 32 - __builtin_clz(spread[w]) : 0; };
    const bool v2 = (reinterpret_cast<uintptr_t>(io.bkeys) & 7) == 0;
    // MSD fast path: one stable sort (records start in record order) by a
    // 64-bit digit packing the most significant varying key bits above the
    // action bit, i.e. by (top key bits, action, record). If no two
    // neighbours share those key bits without sharing the whole key (checked
    // on the device), the order is already the final (key, action, record)
    // order; otherwise fall back to the full LSD below. Typical keys differ
    // within their first varying words, so one sort replaces the action pass
    // plus ceil(varying bits / 64) key passes, and the action travels in the
    // sorted digit instead of being gathered per record afterwards. The
    // packing comes from the sample; the first pass reports the exact spread,
    // and a packing that missed a varying bit (of a packed word, of a word
    // before the last packed one, or of the action) is re-run with it.
    bool resolved = false;
    for (int attempt = 0; attempt < 2; ++attempt) {
        const int abits = bits_of(KW) > 0 ? 1 : 0;
        int ws[8], bs[8], nf = 0, used = abits, w = 0;
        for (; w < KW && nf + abits < 8; ++w) {
            const int b = bits_of(w);
            if (b == 0) continue;
            if (used + b > 64) break;
            ws[nf] = w;
            bs[nf] = b;
            ++nf;
            used += b;
        }
        int w_rest = w;
        while (w_rest < KW && bits_of(w_rest) == 0) ++w_rest;
        WordPack wp{};
        {
            int off = used;
            for (int f = 0; f < nf; ++f) {  // most significant word in the highest bits
                off -= bs[f];
                wp.mask[ws[f]] = bs[f] >= 32 ? 0xFFFFFFFFu : ((1u << bs[f]) - 1u);
                wp.off[ws[f]] = (uint32_t)off;
            }
            wp.mask[KW] = abits ? 1u : 0u;  // the action: least significant field
        }
        QT_CK(cudaMemsetAsync(exact, 0, sizeof(uint32_t) * (KW + 1), st));
        if (v2)
            qt_first_pass_kernel<true><<<grid, 256, 0, st>>>(v, nrec, wp, reinterpret_cast<unsigned long long*>(io.digit),
                                                             exact, io.reward, io.now, static_cast<ulonglong2*>(io.rn));
        else
            qt_first_pass_kernel<false><<<grid, 256, 0, st>>>(v, nrec, wp, reinterpret_cast<unsigned long long*>(io.digit),
                                                              exact, io.reward, io.now, static_cast<ulonglong2*>(io.rn));
        if (nf > 0) {
            QT_CK(cub::DeviceRadixSort::SortPairs(io.temp, io.temp_bytes,
                                                  reinterpret_cast<const unsigned long long*>(io.digit),
                                                  reinterpret_cast<unsigned long long*>(io.digit2), io.perm,
                                                  io.perm2, (int)nrec, 0, used, st));
            std::swap(io.perm, io.perm2);
            QT_CK(cudaMemsetAsync(io.spread + KW + 1, 0, sizeof(uint32_t), st));
            qt_msd_heads_kernel<<<grid, 256, 0, st>>>(
                v, io.perm, reinterpret_cast<const unsigned long long*>(io.digit2), nrec, w_rest, abits,
                io.spread + KW + 1, io.seg_head, io.key_head);
        }
        uint32_t back[KW + 2];  // unresolved flag, exact spread
        QT_CK(cudaMemcpyAsync(back, io.spread + KW + 1, sizeof(back), cudaMemcpyDeviceToHost, st));
        QT_CK(cudaStreamSynchronize(st));
        bool packing_ok = true;
        for (int x = 0; x < KW; ++x)
            if (x < w_rest && (back[1 + x] & ~wp.mask[x])) packing_ok = false;
        if (back[1 + KW] && !abits) packing_ok = false;
        for (int x = 0; x <= KW; ++x) spread[x] = back[1 + x];  // exact from here on
        if (packing_ok) {
            resolved = nf > 0 && back[0] == 0;
            break;
        }
        qt_iota_kernel<<<grid, 256, 0, st>>>(io.perm, nrec);
    }
    if (!resolved) qt_iota_kernel<<<grid, 256, 0, st>>>(io.perm, nrec);
    // LSD over the packed key: the action is the least significant field, then
    // words 29 .. 0; each pass packs up to 64 bits of varying fields (constant
    // words are skipped: they cannot reorder anything)
    int w_next = resolved ? -1 : KW;  // KW = action, then 29, 28, ..., 0
    while (w_next >= 0) {
        PackSpec ps{};
        int used = 0;
        while (w_next >= 0 && ps.nf < 8) {
            const int w = w_next == KW ? KW : w_next;
            const int b = bits_of(w);
            if (b == 0) {  // constant field
                w_next = w == KW ? KW - 1 : w_next - 1;
                continue;
            }
            if (used + b > 64) break;
            ps.w[ps.nf] = w;
            ps.bits[ps.nf] = b;
            ps.off[ps.nf] = used;
            ps.nf++;
            used += b;
            w_next = w == KW ? KW - 1 : w_next - 1;
        }
        if (ps.nf == 0) break;
        qt_gather_digit_kernel<<<grid, 256, 0, st>>>(v, io.perm, nrec, ps,
                                                     reinterpret_cast<unsigned long long*>(io.digit));
        QT_CK(cub::DeviceRadixSort::SortPairs(io.temp, io.temp_bytes,
                                              reinterpret_cast<const unsigned long long*>(io.digit),
                                              reinterpret_cast<unsigned long long*>(io.digit2), io.perm,
                                              io.perm2, (int)nrec, 0, used, st));
        uint32_t* t = io.perm;
        io.perm = io.perm2;
        io.perm2 = t;
    }
    if (!resolved) qt_heads_kernel<<<grid, 256, 0, st>>>(v, io.perm, nrec, io.seg_head, io.key_head);
    QT_CK(cub::DeviceScan::ExclusiveSum(io.temp, io.temp_bytes, io.seg_head, io.seg_scan, (int)nrec, st));
    QT_CK(cub::DeviceScan::InclusiveSum(io.temp, io.temp_bytes, io.key_head, io.key_scan, (int)nrec, st));
    uint32_t tail[3];
    QT_CK(cudaMemcpyAsync(&tail[0], io.seg_scan + nrec - 1, 4, cudaMemcpyDeviceToHost, st));
    QT_CK(cudaMemcpyAsync(&tail[1], io.seg_head + nrec - 1, 4, cudaMemcpyDeviceToHost, st));
    QT_CK(cudaMemcpyAsync(&tail[2], io.key_scan + nrec - 1, 4, cudaMemcpyDeviceToHost, st));
    QT_CK(cudaStreamSynchronize(st));
    nseg = (size_t)tail[0] + tail[1];
    nkeys = tail[2];
    qt_seg_list_kernel<<<grid, 256, 0, st>>>(io.seg_head, io.seg_scan, io.key_scan, nrec, io.seg_start,
                                             io.seg_key);
    return cudaGetLastError();
}

cudaError_t qt_fold(const QtFoldIO& io, size_t nseg, size_t nkeys, uint32_t* keys, double* q, uint64_t* t,
                    uint64_t* cnt, uint8_t* has, int num_sms, cudaStream_t st) {
    FoldArgs f{};
    f.v = rec_view(io);
    f.perm = io.perm;
    f.nrec = io.n_init + io.n;
    f.nseg = nseg;
    f.seg_start = io.seg_start;
    f.seg_key = io.seg_key;
    f.old_q = io.old_q;
    f.old_t = io.old_t;
    f.old_cnt = io.old_cnt;
    f.rn = reinterpret_cast<const ulonglong2*>(io.rn);
    f.limit = io.limit;
    f.alpha = io.alpha;
    f.omega = io.omega;
    f.keys = keys;
    f.q = q;
    f.t = t;
    f.cnt = cnt;
    f.has = has;
    f.bad = io.bad;
    // the last sort's input digits are dead by now: a [nkeys] u32 scratch
    f.src_rec = io.digit;
    cudaError_t e = cudaMemsetAsync(f.src_rec, 0xFF, sizeof(uint32_t) * nkeys, st);
    if (e != cudaSuccess) return e;
    qt_fold_kernel<<<num_sms * 4, 128, 0, st>>>(f);
    qt_copy_keys_kernel<<<num_sms * 8, 256, 0, st>>>(f.v, f.src_rec, nkeys, keys);
    return cudaGetLastError();
}

}  // namespace gbxcu
