// k_shuffle.cu — device replay of fit's per-epoch in-place Fisher-Yates
// shuffle (proj/src/policy.cpp:303-314), in closed form.
//
// The sequential loop `for i = n..2: j = next_below(i); swap(order[i-1],
// order[j])` is the swap sequence S_p = (p, j_p), p = n-1 down to 1, whose
// partners depend only on the SplitMix64 stream: j_p = umulhi(draw_{n-p}, p+1)
// with draw_k = fin(seed + k*gamma) (skip-ahead). Group swaps by target:
// list(x) = {q : j_q = x} sorted ascending. Position p >= 1 is never touched
// after S_p, and S_p moves into p whatever sat at j_p just before it; the last
// swap to write j_p before S_p is succ(p), the next-larger element of
// list(j_p). What S_q writes into j_q is V(q) = the value at q just before S_q,
// which in turn was written by fg(q) = min{q' > q : j_q' = q}. Hence
//   V(q)     = A[root(q)],  root = end of the chain q -> fg(q) -> fg(fg(q)) ...
//   final[p] = succ(p) ? V(succ(p)) : A[j_p]            (p >= 1)
//   final[0] = fg(0)   ? V(fg(0))   : A[0]
// Chains are O(log n) long (pointer jumping would need ~6 rounds at n = 1e6
// and 1e7; buckets hold <= ~21 swaps), so each thread walks its own chain
// end in one pass, instead of the O(log n) *dependence depth* of ~50 rounds a
// reservation-based replay needs. The
// result equals the sequential shuffle exactly (tests/test_gpu_parity.py
// compares against the reference at 1e5 and 1e6).
#include "common.cuh"
#include "kernels.h"

namespace gbxcu {

constexpr uint32_t NONE = 0xFFFFFFFFu;
constexpr int LOCAL_BUCKET = 32;

__global__ void iota_kernel(uint32_t* __restrict__ order, size_t n) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x)
        order[i] = (uint32_t)i;
}

__device__ __forceinline__ uint32_t partner(uint64_t seed_e, uint32_t n, uint32_t p) {
    return (uint32_t)below_of(sm_draw(seed_e, (uint64_t)(n - p)), (uint64_t)p + 1);
}

__global__ void __launch_bounds__(SHUF_BLOCK)
shuffle_epoch_kernel(ShuffleArgs s) {
    if (*s.diverged >= 0) return;
    unsigned int target = 0;
    const uint32_t n = s.n;
    const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t nthr = (size_t)gridDim.x * blockDim.x;

    // 1: empty buckets
    for (size_t x = tid; x < n; x += nthr) __stcg(s.head + x, NONE);
    grid_barrier(s.bar, target);

    // 2: partners + bucket lists (arbitrary order inside a bucket)
    for (size_t p = tid + 1; p < n; p += nthr) {
        const uint32_t j = partner(s.seed_e, n, (uint32_t)p);
        __stcg(s.jp + p, j);
        __stcg(s.nxt + p, atomicExch(s.head + j, (uint32_t)p));
    }
    grid_barrier(s.bar, target);

    // 3: sort each bucket -> succ() of its members, fg(x), chain start
    for (size_t x = tid; x < n; x += nthr) {
        uint32_t loc[LOCAL_BUCKET];
        int m = 0;
        bool overflow = false;
        for (uint32_t e = __ldcg(s.head + x); e != NONE; e = __ldcg(s.nxt + e)) {
            if (m < LOCAL_BUCKET) loc[m] = e;
            else overflow = true;
            ++m;
        }
        uint32_t fg = NONE;
        if (!overflow) {
            for (int a = 1; a < m; ++a) {  // insertion sort, ascending
                const uint32_t v = loc[a];
                int b = a - 1;
                while (b >= 0 && loc[b] > v) { loc[b + 1] = loc[b]; --b; }
                loc[b + 1] = v;
            }
            for (int k = 0; k < m; ++k) {
                __stcg(s.succ + loc[k], k + 1 < m ? loc[k + 1] : NONE);
                if (fg == NONE && loc[k] > x) fg = loc[k];
            }
        } else {
            // rare (> 32 swaps aimed at one slot): quadratic walk of the list
            for (uint32_t e = __ldcg(s.head + x); e != NONE; e = __ldcg(s.nxt + e)) {
                uint32_t nx = NONE;
                for (uint32_t f = __ldcg(s.head + x); f != NONE; f = __ldcg(s.nxt + f))
                    if (f > e && f < nx) nx = f;
                __stcg(s.succ + e, nx);
                if (e > x && e < fg) fg = e;
            }
        }
        __stcg(s.root + x, fg != NONE ? fg : (uint32_t)x);
        if (x == 0) __stcg(s.fg0, fg);
    }
    grid_barrier(s.bar, target);

    // 4: chain ends, walked directly: fg() strictly increases along a chain,
    //    so each walk terminates; chains are O(log n) long (expected ~1-2, the
    //    longest a few dozen), so one pass of dependent L2 loads replaces the
    //    ~7 barrier-separated pointer-jumping rounds (half of the kernel's time)
    for (size_t q = tid; q < n; q += nthr) {
        uint32_t r = __ldcg(s.root + q);
        if (r != (uint32_t)q) {
            for (uint32_t r2 = __ldcg(s.root + r); r2 != r; r2 = __ldcg(s.root + r)) r = r2;
        }
        __stcg(s.root2 + q, r);
    }
    grid_barrier(s.bar, target);
    const uint32_t* cur = s.root2;

    // 5: final permutation
    const uint32_t fg0 = __ldcg(s.fg0);
    for (size_t p = tid; p < n; p += nthr) {
        uint32_t src;
        if (p == 0) {
            src = fg0 != NONE ? __ldcg(cur + fg0) : 0u;
        } else {
            const uint32_t sc = __ldcg(s.succ + p);
            src = sc != NONE ? __ldcg(cur + sc) : __ldcg(s.jp + p);
        }
        s.out[p] = __ldg(s.in + src);
    }
}

}  // namespace gbxcu
