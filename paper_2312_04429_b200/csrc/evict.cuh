// evict.cuh -- device helpers of the eviction kernels (kernels.cu: the radix-select building
// blocks of the distributed protocol; evict.cu: the fused single-cache select + apply).
#pragma once
#include "common.cuh"

namespace nv {

// Policy score of item (e, j) (CACHE_POLICY_*): LCBFU f*K, LRU last-access clock,
// LFU f, FIFO 0 (the id decides).  Item key: min(score, 2^29-1) << 35 | id << 3 | j.
// Entry key (R24): the policy score aggregated over the entry's stored items (LCBFU sum f*K,
// LFU sum f, LRU max last access, FIFO 0), min(., 2^32-1) << 32 | id.
// The kernels are instantiated per (policy, granularity) with the K values in registers: a
// runtime switch and constant-bank loads per item made the sweep instruction-bound (ncu r1y:
// ~120 SASS instructions per item, 68% issue-slot use at 1.1 TB/s).
template <int POLICY>
__device__ __forceinline__ unsigned long long item_score(const uint32_t* __restrict__ fcnt,
                                                         const uint32_t* __restrict__ lastacc, int64_t it, int kvj) {
    if constexpr (POLICY == CACHE_POLICY_LRU) return lastacc[it];
    else if constexpr (POLICY == CACHE_POLICY_LFU) return fcnt[it];
    else if constexpr (POLICY == CACHE_POLICY_FIFO) return 0ull;
    else return (unsigned long long)fcnt[it] * (unsigned long long)(unsigned)kvj;
}

__device__ __forceinline__ unsigned long long item_key(unsigned long long sc, uint32_t id, int j) {
    if (sc > 0x1FFFFFFFull) sc = 0x1FFFFFFFull;
    return (sc << 35) | ((unsigned long long)id << 3) | (unsigned long long)j;
}

template <int POLICY>
__device__ __forceinline__ unsigned long long entry_key(const uint32_t* __restrict__ fcnt,
                                                        const uint32_t* __restrict__ lastacc, int64_t e, uint32_t m,
                                                        uint32_t id, int nk, const int (&kv)[CACHE_MAX_K]) {
    unsigned long long sc = 0ull;
#pragma unroll
    for (int j = 0; j < CACHE_MAX_K; ++j) {
        if (j >= nk || !((m >> j) & 1u)) continue;
        const unsigned long long v = item_score<POLICY>(fcnt, lastacc, e * nk + j, kv[j]);
        if constexpr (POLICY == CACHE_POLICY_LRU) sc = v > sc ? v : sc;
        else sc += v;
    }
    if (sc > 0xFFFFFFFFull) sc = 0xFFFFFFFFull;
    return (sc << 32) | (unsigned long long)id;
}

// Per-thread run-length aggregation of histogram increments: consecutive keys of a thread
// mostly share a digit (early passes: almost all), so one shared atomic per run.
struct DigitRun {
    unsigned cur = 0xFFFFFFFFu, cnt = 0;
    __device__ __forceinline__ void add(unsigned* sh, unsigned d) {
        if (d == cur) { ++cnt; return; }
        if (cnt) atomicAdd(&sh[cur], cnt);
        cur = d;
        cnt = 1;
    }
    __device__ __forceinline__ void add_n(unsigned* sh, unsigned d, unsigned n) {
        if (d == cur) { cnt += n; return; }
        if (cnt) atomicAdd(&sh[cur], cnt);
        cur = d;
        cnt = n;
    }
    __device__ __forceinline__ void flush(unsigned* sh) {
        if (cnt) atomicAdd(&sh[cur], cnt);
    }
};

// One output slot range per warp and key column: a ballot of the evicting lanes, one atomic by
// the leader, each lane's index = its rank among them (per-lane atomics on one counter
// serialised at L2).  Item mode also emits each item's entry slot so the host updates its
// mirrors without an id lookup.  The sweep is warp-uniform (lane l takes slot base + l).
__device__ __forceinline__ unsigned long long warp_claim(unsigned long long* counter, bool take, int lane) {
    const unsigned bal = __ballot_sync(0xFFFFFFFFu, take);
    unsigned long long base = 0;
    if (bal) {
        if (lane == __ffs(bal) - 1) base = atomicAdd(counter, (unsigned long long)__popc(bal));
        base = __shfl_sync(0xFFFFFFFFu, base, __ffs(bal) - 1);
    }
    return base + (unsigned long long)__popc(bal & ((1u << lane) - 1u));
}


// Instantiate KERN(policy, granularity) for the runtime (km.policy, km.gran).
#define NV_EVICT_DISPATCH(KERN, ...)                                                                   \
    do {                                                                                               \
        const int pol_ = km.policy, gr_ = km.gran;                                                     \
        if (gr_ == CACHE_EVICT_ENTRY) {                                                                \
            if (pol_ == CACHE_POLICY_LRU) KERN(CACHE_POLICY_LRU, CACHE_EVICT_ENTRY);                   \
            else if (pol_ == CACHE_POLICY_LFU) KERN(CACHE_POLICY_LFU, CACHE_EVICT_ENTRY);              \
            else if (pol_ == CACHE_POLICY_FIFO) KERN(CACHE_POLICY_FIFO, CACHE_EVICT_ENTRY);            \
            else KERN(CACHE_POLICY_LCBFU, CACHE_EVICT_ENTRY);                                          \
        } else {                                                                                       \
            if (pol_ == CACHE_POLICY_LRU) KERN(CACHE_POLICY_LRU, CACHE_EVICT_ITEM);                    \
            else if (pol_ == CACHE_POLICY_LFU) KERN(CACHE_POLICY_LFU, CACHE_EVICT_ITEM);               \
            else if (pol_ == CACHE_POLICY_FIFO) KERN(CACHE_POLICY_FIFO, CACHE_EVICT_ITEM);             \
            else KERN(CACHE_POLICY_LCBFU, CACHE_EVICT_ITEM);                                           \
        }                                                                                              \
    } while (0)

}  // namespace nv
