// k_shuffle.cu — device replay of fit's per-epoch in-place Fisher-Yates
// shuffle (proj/src/policy.cpp:303-314).
//
// The sequential loop `for i = n..2: j = next_below(i); swap(order[i-1],
// order[j])` is a fixed sequence of swaps S_p = (p, j_p), p = n-1..1, whose
// partners depend only on the stream: j_p = umulhi(draw_{n-p}, p+1) with
// draw_k = fin(seed + k*gamma) (SplitMix64 skip-ahead). Swaps on disjoint
// positions commute, so S can be applied out of order as long as, per
// position, swaps land in sequence order. Deterministic reservations
// (Shun, Blelloch, Fineman, Gibbons, SODA'15): every pending swap
// atomicMax-reserves its two positions with priority p (earlier swap = larger
// p); a swap commits when it holds both reservations. The earliest pending
// swap always commits, the committed set touches disjoint positions, and the
// result equals the sequential shuffle exactly. Dependence depth is O(log n)
// w.h.p., so an epoch's permutation takes a few dozen rounds of one
// persistent cooperative kernel instead of n serial host steps.
#include "common.cuh"
#include "kernels.h"

namespace gbxcu {

__global__ void iota_kernel(uint32_t* __restrict__ order, size_t n) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x)
        order[i] = (uint32_t)i;
}

__device__ __forceinline__ uint32_t partner(uint64_t seed_e, uint32_t n, uint32_t p) {
    return (uint32_t)below_of(sm_draw(seed_e, (uint64_t)(n - p)), (uint64_t)p + 1);
}

// resv[] must be all -1 on entry and is left all -1 on exit.
// counters[0..1]: list lengths (counters[0] = 0 on entry), counters[2] scratch.
__global__ void __launch_bounds__(SHUF_BLOCK)
shuffle_epoch_kernel(uint32_t* __restrict__ order, uint32_t n, uint64_t seed_e,
                     int* __restrict__ resv, uint32_t* __restrict__ list_a,
                     uint32_t* __restrict__ list_b, unsigned int* __restrict__ counters,
                     unsigned int* __restrict__ bar, const int* __restrict__ diverged) {
    if (*diverged >= 0 || n < 2) return;
    unsigned int target = 0;
    const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t nthr = (size_t)gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31;

    // pending list: every swap position p = 1..n-1
    for (size_t t = tid; t < (size_t)n - 1; t += nthr) list_a[t] = (uint32_t)(t + 1);
    if (tid == 0) {
        counters[0] = n - 1;
        counters[1] = 0;
    }
    grid_barrier(bar, target);

    uint32_t* cur = list_a;
    uint32_t* nxt = list_b;
    int ci = 0;
    for (;;) {
        const unsigned int cnt = __ldcg(counters + ci);
        if (cnt == 0) break;
        // reserve
        for (size_t t = tid; t < cnt; t += nthr) {
            const uint32_t p = __ldcg(cur + t);
            const uint32_t j = partner(seed_e, n, p);
            atomicMax(resv + p, (int)p);
            if (j != p) atomicMax(resv + j, (int)p);
        }
        grid_barrier(bar, target);
        // commit or carry over
        const size_t cnt_round = ((cnt + nthr - 1) / nthr) * nthr;  // warp-uniform trip count
        for (size_t t = tid; t < cnt_round; t += nthr) {
            bool carry = false;
            uint32_t p = 0;
            if (t < cnt) {
                p = __ldcg(cur + t);
                const uint32_t j = partner(seed_e, n, p);
                const bool win = __ldcg(resv + p) == (int)p && __ldcg(resv + j) == (int)p;
                if (win) {
                    if (j != p) {
                        const uint32_t a = __ldcg(order + p), b = __ldcg(order + j);
                        __stcg(order + p, b);
                        __stcg(order + j, a);
                    }
                } else {
                    carry = true;
                }
            }
            const unsigned int m = __ballot_sync(0xffffffffu, carry);
            if (m) {
                unsigned int base = 0;
                if (lane == 0) base = atomicAdd(counters + (ci ^ 1), __popc(m));
                base = __shfl_sync(0xffffffffu, base, 0);
                if (carry) __stcg(nxt + base + __popc(m & ((1u << lane) - 1)), p);
            }
        }
        grid_barrier(bar, target);
        // release reservations of this round
        for (size_t t = tid; t < cnt; t += nthr) {
            const uint32_t p = __ldcg(cur + t);
            const uint32_t j = partner(seed_e, n, p);
            __stcg(resv + p, -1);
            __stcg(resv + j, -1);
        }
        if (tid == 0) counters[ci] = 0;
        grid_barrier(bar, target);
        uint32_t* tmp = cur;
        cur = nxt;
        nxt = tmp;
        ci ^= 1;
    }
}

}  // namespace gbxcu
