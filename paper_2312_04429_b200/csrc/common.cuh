// common.cuh -- internal helpers of the B200 NIRVANA cache library (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "../../include/nirvana_cache.h"

namespace nv {

constexpr int kTileN = 256;          // entry-slot padding granularity (one tcgen05 N tile)
constexpr int kMaxDim = 1024;

// ---------------------------------------------------------------------------------------
// Ranking key.  Total order of a candidate (t, id): t descending, then id ascending
// (reading R3).  t is the fp32 scan value fl(<q~,x~> * inv_norm(x~)); -0.0 is canonicalised
// to +0.0 so equal scores compare equal.  key = orderable(t) << 32 | (0xFFFFFFFF - id):
// a larger key is a better candidate; key 0 means "no candidate".
// ---------------------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint32_t orderable_f32(float t) {
    uint32_t u;
#ifdef __CUDA_ARCH__
    u = __float_as_uint(t);
#else
    memcpy(&u, &t, 4);
#endif
    if (u == 0x80000000u) u = 0u;
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__host__ __device__ __forceinline__ float key_to_f32(unsigned long long key) {
    uint32_t o = (uint32_t)(key >> 32);
    uint32_t u = (o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o;
#ifdef __CUDA_ARCH__
    return __uint_as_float(u);
#else
    float f;
    memcpy(&f, &u, 4);
    return f;
#endif
}

__host__ __device__ __forceinline__ unsigned long long make_key(float t, uint32_t id) {
    return ((unsigned long long)orderable_f32(t) << 32) | (unsigned long long)(0xFFFFFFFFu - id);
}

__host__ __device__ __forceinline__ uint32_t key_id(unsigned long long key) {
    return 0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFull);
}

// One partial top-k record written by a scoring kernel: 16 bytes.
struct __align__(16) Rec {
    unsigned long long key;
    uint32_t slot;
    uint32_t pad;
};

// Register-resident running top-k of one query (sorted, best first).  KMAX is a compile-time
// bound; entries beyond the requested topk are simply never read.
template <int KMAX>
struct TopK {
    unsigned long long k[KMAX];
    uint32_t s[KMAX];
    float thr;   // scan value of the current KMAX-th best (-inf while not full)

    __device__ __forceinline__ void init() {
#pragma unroll
        for (int i = 0; i < KMAX; ++i) { k[i] = 0ull; s[i] = 0xFFFFFFFFu; }
        thr = -INFINITY;
    }
    // Offer a candidate with a precomputed key (key must be > 0).
    __device__ __forceinline__ void offer_key(unsigned long long key, uint32_t slot) {
        if (key <= k[KMAX - 1]) return;
#pragma unroll
        for (int i = KMAX - 1; i > 0; --i) {
            if (key > k[i - 1]) { k[i] = k[i - 1]; s[i] = s[i - 1]; }
            else if (key > k[i]) { k[i] = key; s[i] = slot; }
        }
        if (key > k[0]) { k[0] = key; s[0] = slot; }
        if (k[KMAX - 1] != 0ull) thr = fmaxf(thr, key_to_f32(k[KMAX - 1]));   // thr may carry an outside bound
    }
    // Offer scan value t of entry slot `slot`; the id is loaded only when t can enter.
    __device__ __forceinline__ void offer(float t, uint32_t slot, const uint32_t* __restrict__ ids) {
        if (!(t >= thr)) return;       // also rejects NaN (invalid slots carry inv_norm = NaN)
        offer_key(make_key(t, __ldg(ids + slot)), slot);
    }
    // Remove the best element (shift left); used by warp merges.
    __device__ __forceinline__ void pop() {
#pragma unroll
        for (int i = 0; i < KMAX - 1; ++i) { k[i] = k[i + 1]; s[i] = s[i + 1]; }
        k[KMAX - 1] = 0ull;
        s[KMAX - 1] = 0xFFFFFFFFu;
    }
};

__device__ __forceinline__ unsigned long long shfl_xor_u64(unsigned long long v, int m) {
    uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
    lo = __shfl_xor_sync(0xFFFFFFFFu, lo, m);
    hi = __shfl_xor_sync(0xFFFFFFFFu, hi, m);
    return ((unsigned long long)hi << 32) | lo;
}

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
        unsigned long long o = shfl_xor_u64(v, m);
        v = o > v ? o : v;
    }
    return v;
}

// Query-time constants of the Fig. 11 map passed by value to kernels.
struct KMap {
    double thr[CACHE_MAX_K];
    int32_t kv[CACHE_MAX_K];
    int32_t num_k;
    int32_t k_bias;
    int32_t policy;   // CACHE_POLICY_* (eviction kernels)
    int32_t gran;     // CACHE_EVICT_ITEM / CACHE_EVICT_ENTRY
};

}  // namespace nv
