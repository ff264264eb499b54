// evict.cu -- fused single-cache eviction (readings R11-R13, R24).
//
// cache_evict(n) removes the n units (items, or whole entries in entry mode) with the smallest
// unit keys (evict.cuh: policy score << 35 | id << 3 | j, or aggregated score << 32 | id).
// Keys are unique, so "the n smallest" is exact.  Round 1 ran an 8-pass MSB radix select:
// 8 full sweeps of the slot columns (28 B per slot each) + an apply sweep, 17 launches, and
// ~8-10x its traffic floor at 12.5M entries.  This kernel does the whole selection and the
// apply in ONE cooperative launch with (normally) two full sweeps:
//
//   level 0  full sweep: histogram of every live key over 4,096 LOG bins (keys < 64 exact,
//            else 6 exponent bits + the 6 bits below the leading one) -- monotone in the key
//            and fine where the distribution is dense near its minimum (never-accessed items:
//            score 0, key = id << 3 | j); the min key is reduced alongside (the sort base).
//   pick     every CTA scans the global histogram (same result everywhere, no extra sync):
//            bin b holding the n-th smallest key -> range [lo, lo + 2^w), rank r inside it.
//   level l  linear 12-bit digits of (key - lo).  A FULL sweep also applies every unit with
//            key < lo (certain to go) and, when the range's count fits the candidate buffer,
//            compacts the range's (key, slot) pairs; after that the levels sweep only the
//            candidates.  Stops as soon as the chosen range holds exactly r keys (or w = 0):
//            threshold T = lo + 2^w - 1.
//   apply    the candidates with key <= T (or, without compaction, one more full sweep):
//            presence bit cleared (atomicAnd: the last bit of an entry makes it dirty),
//            counter reset, latent slot listed, dirty entry invalidated (inv_norm = NaN).
//
// Grid = one resident wave (cooperative launch; grid.sync between levels).  Histograms live
// in distinct per-level buffers, so no level re-zeroes a buffer another CTA may still read.
#include <cooperative_groups.h>

#include "kernels.h"
#include "evict.cuh"

namespace nv {

namespace cg = cooperative_groups;

#ifndef NV_SEL_CPASYNC
#define NV_SEL_CPASYNC 0   // 1: |K| = 5 sweeps fed by per-lane cp.async rings (measured slower, kept for the record)
#endif
constexpr bool kSelCpAsync = NV_SEL_CPASYNC != 0;
#ifndef NV_SEL_PREFETCH
#define NV_SEL_PREFETCH 0   // 1: next group's loads issued before this group's work (measured: no gain)
#endif
constexpr bool kSelPrefetch = NV_SEL_PREFETCH != 0 && !kSelCpAsync;
#ifndef NV_SEL_COLT
#define NV_SEL_COLT 0   // 1: coalesced column loads + shared-memory redistribution (measured: no gain)
#endif
constexpr bool kSelColT = NV_SEL_COLT != 0;
#ifndef NV_SEL_DYN_PCT
#define NV_SEL_DYN_PCT 25  // the last 25% of each full sweep's groups are claimed dynamically (two-sweep path: 275-311 -> 227-228 us at 12.5M; the window path: no change)
#endif
constexpr int kSelDynPct = NV_SEL_DYN_PCT;
constexpr int kColTBytes = (kSelCpAsync ? 256 : 512) / 32 * 160 * 16;   // per-warp 2,560-B transposes
constexpr int kSelThreads = (kSelCpAsync || kSelPrefetch) ? 256 : 512;
constexpr int kCpStages = 3;                           // groups per lane: 2 loading + 1 being processed
constexpr int kCpRingBytes = kCpStages * kSelThreads * 112;

// NV_SEL_TRACE=1 (experiments only): every CTA's thread 0 stamps %globaltimer at each phase
// boundary of the fused kernel; per stamp index the earliest and latest CTA are kept
// (cache_debug_sel_trace), so a phase's cost and its slowest-CTA tail can be read apart.
#ifndef NV_SEL_TRACE
#define NV_SEL_TRACE 0
#endif
__device__ unsigned long long g_sel_tmin[kSelTraceN], g_sel_tmax[kSelTraceN];
__device__ unsigned long long g_sel_cta[kSelTraceCta][1024];   // the first stamps, per CTA
__device__ __forceinline__ void sel_stamp(int& i) {
    if constexpr (NV_SEL_TRACE != 0) {
        if (threadIdx.x == 0 && i < kSelTraceN) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            atomicMin(&g_sel_tmin[i], t);
            atomicMax(&g_sel_tmax[i], t);
            if (i < kSelTraceCta && blockIdx.x < 1024) g_sel_cta[i][blockIdx.x] = t;
        }
        ++i;
    }
}

__device__ __forceinline__ uint32_t sel_bin0(unsigned long long key) {
    if (key < 64ull) return (uint32_t)key;
    const int e = 63 - __clzll((long long)key);   // 6..63
    return 64u + (uint32_t)(e - 6) * 64u + (uint32_t)((key >> (e - 6)) & 63ull);
}
// range of level-0 bin b: [lo, lo + 2^w)
__device__ __forceinline__ void sel_bin0_range(uint32_t b, unsigned long long& lo, int& w) {
    if (b < 64u) { lo = b; w = 0; return; }
    const int e = (int)((b - 64u) >> 6) + 6, m = (int)((b - 64u) & 63u);
    w = e - 6;
    lo = (unsigned long long)(64 + m) << w;
}

// Every CTA: find the bin holding the target-th (1-based) key of histogram h.  Returns the
// bin (kSelBins if the histogram holds fewer keys: an inconsistent live count), the number
// of keys in lower bins and the bin's count.
struct PickRes {
    uint32_t bin;
    unsigned long long before, cnt;
};
__device__ PickRes sel_pick(const uint32_t* h, unsigned long long target) {
    __shared__ unsigned long long s_w[kSelThreads / 32];
    __shared__ PickRes s_res;
    constexpr int PER = kSelBins / kSelThreads;   // 8 or 16 bins per thread
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    uint32_t v[PER];
    const uint4* h4 = reinterpret_cast<const uint4*>(h + t * PER);
#pragma unroll
    for (int q = 0; q < PER / 4; ++q) {
        const uint4 x4 = __ldcg(h4 + q);
        v[4 * q] = x4.x; v[4 * q + 1] = x4.y; v[4 * q + 2] = x4.z; v[4 * q + 3] = x4.w;
    }
    unsigned long long s = 0;
#pragma unroll
    for (int i = 0; i < PER; ++i) s += v[i];
    unsigned long long x = s;   // inclusive scan over the block
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= o) x += y;
    }
    if (t == 0) s_res = PickRes{(uint32_t)kSelBins, 0ull, 0ull};
    if (lane == 31) s_w[w] = x;
    __syncthreads();
    unsigned long long off = 0;
    for (int i = 0; i < w; ++i) off += s_w[i];
    const unsigned long long excl = off + x - s;
    if (excl < target && target <= excl + s) {
        unsigned long long c = excl;
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            if (c + v[i] >= target) { s_res = PickRes{(uint32_t)(t * PER + i), c, v[i]}; break; }
            c += v[i];
        }
    }
    __syncthreads();
    const PickRes r = s_res;
    __syncthreads();   // s_res / s_w are reused by the next pick
    return r;
}

// Every CTA: the number of keys in histogram h.
__device__ unsigned long long sel_total(const uint32_t* h) {
    __shared__ unsigned long long s_t[kSelThreads / 32];
    unsigned long long x = 0;
    for (int i = threadIdx.x; i < kSelBins; i += kSelThreads) x += __ldcg(h + i);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) x += __shfl_xor_sync(0xFFFFFFFFu, x, o);
    if ((threadIdx.x & 31) == 0) s_t[threadIdx.x >> 5] = x;
    __syncthreads();
    unsigned long long t = 0;
    for (int i = 0; i < kSelThreads / 32; ++i) t += s_t[i];
    __syncthreads();
    return t;
}

// Sweep modes (uniform over the grid within a phase)
enum { kSweepL0 = 0, kSweepLevel = 1, kSweepFinal = 2 };

struct SelLevel {
    unsigned long long lo, T;
    int w, shift;          // range [lo, lo + 2^w); digit = (key - lo) >> shift
    bool compact;
    unsigned long long kb, ev_lim;   // evicted-key bitmap over [kb, kb + ev_lim) (ev_lim 0: off)
};

// Evicted keys are also marked, as they are evicted, in a bitmap over [min key, min key +
// 32 x words): when none falls beyond it the kernel emits the list sorted by an ordered
// compaction (keys are unique).  One atomic per (lane, word) run.
struct BitRun {
    long long w = -1;
    uint32_t m = 0u;
    __device__ __forceinline__ void add(const SelArgs& a, const SelLevel& L, unsigned long long key) {
        if (!L.ev_lim) return;
        const unsigned long long d = key - L.kb;
        if (d >= L.ev_lim) { atomicExch(&a.out->ev_over, 1u); return; }   // overflow: sort on the host side
        const long long ww = (long long)(d >> 5);
        if (ww != w) { flush(a); w = ww; }
        m |= 1u << (d & 31);
    }
    __device__ __forceinline__ void flush(const SelArgs& a) {
        if (m) atomicOr(a.ev_bits + w, m);
        m = 0u;
    }
};
__device__ __forceinline__ void ev_mark(const SelArgs& a, const SelLevel& L, unsigned long long key) {
    BitRun r;
    r.add(a, L, key);
    r.flush(a);
}

template <int POLICY, int GRAN>
__device__ __forceinline__ void sel_unit_common(const SelArgs& a, int mode, const SelLevel& L,
                                                unsigned long long key, bool live, uint32_t slot,
                                                unsigned* sh, DigitRun& run, unsigned long long& kmin, int lane,
                                                bool& ev) {
    ev = false;
    if (mode == kSweepL0) {
        if (live) {
            run.add(sh, sel_bin0(key));
            kmin = key < kmin ? key : kmin;
        }
        if (L.compact) {   // warp-uniform: the single-sweep window, every key < L.T
            const bool inw = live && key < L.T;
            const unsigned long long at = warp_claim(&a.out->cnt_w, inw, lane);
            if (inw && at < a.cand_cap) { a.cand_key[at] = key; a.cand_slot[at] = slot; }
        }
        return;
    }
    ev = live && (mode == kSweepFinal ? key <= L.T : key < L.lo);
    const bool inr = mode == kSweepLevel && live && !ev && ((key - L.lo) >> L.w) == 0ull;
    if (inr) run.add(sh, (unsigned)((key - L.lo) >> L.shift));
    if (mode == kSweepLevel && L.compact) {   // warp-uniform
        const unsigned long long at = warp_claim(&a.out->cnt[3], inr, lane);
        if (inr && at < a.cand_cap) { a.cand_key[at] = key; a.cand_slot[at] = slot; }
    }
}

// Policy score of an item from its preloaded column value (fcnt for LCBFU / LFU, lastacc for
// LRU, nothing for FIFO) -- the same scores as evict.cuh's item_score / entry_key.
template <int POLICY>
__device__ __forceinline__ unsigned long long score_v(uint32_t col, int kvj) {
    if constexpr (POLICY == CACHE_POLICY_LRU || POLICY == CACHE_POLICY_LFU) return col;
    else if constexpr (POLICY == CACHE_POLICY_FIFO) return 0ull;
    else return (unsigned long long)col * (unsigned long long)(unsigned)kvj;
}

// Dirty entries and freed pool slots are marked in bitmaps (compacted in index order at the
// end of the kernel: the host's free lists and the API's ascending dirty-id list need sorted
// lists, and an ordered compaction of a bitmap is far cheaper than sorting them).
__device__ __forceinline__ void mark_dirty(const SelArgs& a, int64_t e, uint32_t id) {
    atomicOr(a.dslot_bits + (e >> 5), 1u << (e & 31));
    const uint32_t x = id / (uint32_t)a.world;   // ids of this rank: id % world == rank
    atomicOr(a.did_bits + (x >> 5), 1u << (x & 31));
}
__device__ __forceinline__ void mark_pool(const SelArgs& a, int32_t slot) {
    if (a.pool_bits && slot >= 0) atomicOr(a.pool_bits + (slot >> 5), 1u << (slot & 31));
}

// Per-lane run of bits in one bitmap word (one atomic per word change); the final flush is
// warp-collective and ORs the words of neighbouring lanes first (a segmented reduction over
// contiguous lanes with the same word), so the common case -- consecutive slots, ids and pool
// slots across the warp -- costs one atomic per word instead of up to 32 same-address atomics.
struct WordRun {
    uint32_t w = 0xFFFFFFFFu, m = 0u;   // word index < 2^27 (32-bit ids / slots)
    __device__ __forceinline__ void add(uint32_t* bits, uint32_t i) {
        const uint32_t ww = i >> 5;
        if (ww != w) {
            if (m) atomicOr(bits + w, m);
            w = ww;
            m = 0u;
        }
        m |= 1u << (i & 31);
    }
    __device__ __forceinline__ void warp_flush(uint32_t* bits, int lane) {   // all 32 lanes, converged
        const uint32_t mw = m ? w : 0xFFFFFFFFu;
        uint32_t acc = m;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t ow = __shfl_down_sync(0xFFFFFFFFu, mw, o);
            const uint32_t om = __shfl_down_sync(0xFFFFFFFFu, acc, o);
            if (lane + o < 32 && ow == mw) acc |= om;
        }
        const uint32_t pw = __shfl_up_sync(0xFFFFFFFFu, mw, 1);
        if (m && (lane == 0 || pw != mw)) atomicOr(bits + w, acc);
        m = 0u;
        w = 0xFFFFFFFFu;
    }
};

// One entry slot (lane-parallel, warp-uniform control flow), every mode of a full sweep, from
// the slot's preloaded presence mask, id and policy column (col[j] for j < nk).
template <int POLICY, int GRAN>
__device__ __forceinline__ void sel_slot(const SelArgs& a, int nk, const int (&kv)[CACHE_MAX_K], int mode,
                                         const SelLevel& L, int64_t e, uint32_t m, uint32_t id,
                                         const uint32_t (&col)[CACHE_MAX_K], unsigned* sh, DigitRun& run,
                                         unsigned long long& kmin, int lane) {
    if constexpr (GRAN == CACHE_EVICT_ENTRY) {
        unsigned long long sc = 0ull;
#pragma unroll
        for (int j = 0; j < CACHE_MAX_K; ++j) {
            if (j >= nk || !((m >> j) & 1u)) continue;
            const unsigned long long v = score_v<POLICY>(col[j], kv[j]);
            if constexpr (POLICY == CACHE_POLICY_LRU) sc = v > sc ? v : sc;
            else sc += v;
        }
        if (sc > 0xFFFFFFFFull) sc = 0xFFFFFFFFull;
        const unsigned long long key = m ? ((sc << 32) | (unsigned long long)id) : 0ull;
        bool ev;
        sel_unit_common<POLICY, GRAN>(a, mode, L, key, m != 0u, (uint32_t)e, sh, run, kmin, lane, ev);
        if (mode == kSweepL0) return;
        const unsigned long long at = warp_claim(&a.out->cnt[0], ev, lane);
        (void)warp_claim(&a.out->cnt[1], ev, lane);   // dirty count = evicted count in entry mode
        if (ev) {
            atomicAdd(&a.out->cnt[2], (unsigned long long)__popc(m));   // stored states freed
            for (int j = 0; j < nk; ++j) {
                if ((m >> j) & 1u) mark_pool(a, a.lslot[e * nk + j]);
                a.fcnt[e * nk + j] = 0u;
            }
            a.present[e] = 0u;
            a.inv_e[e] = __int_as_float(0x7FC00000);
            mark_dirty(a, e, id);
            if (at < a.ev_cap) a.ev_key[at] = key;
            ev_mark(a, L, key);
        }
    } else {
        uint32_t keep = m;
#pragma unroll
        for (int j = 0; j < CACHE_MAX_K; ++j) {
            if (j >= nk) break;   // warp-uniform
            const bool has = (m >> j) & 1u;
            const unsigned long long key = has ? item_key(score_v<POLICY>(col[j], kv[j]), id, j) : 0ull;
            bool ev;
            sel_unit_common<POLICY, GRAN>(a, mode, L, key, has, (uint32_t)e, sh, run, kmin, lane, ev);
            if (mode == kSweepL0) continue;
            const unsigned long long at = warp_claim(&a.out->cnt[0], ev, lane);
            if (ev) {
                keep &= ~(1u << j);
                if (at < a.ev_cap) a.ev_key[at] = key;
                ev_mark(a, L, key);
                mark_pool(a, a.lslot[e * nk + j]);
                a.fcnt[e * nk + j] = 0u;
            }
        }
        if (mode == kSweepL0) return;
        const bool dirty = m && keep == 0u;
        if (keep != m) {
            a.present[e] = keep;
            if (dirty) {
                a.inv_e[e] = __int_as_float(0x7FC00000);
                mark_dirty(a, e, id);
            }
        }
        (void)warp_claim(&a.out->cnt[1], dirty, lane);
    }
}

// ---- item mode, |K| = 5, 4 slots per lane (the common case, C2-C5) ----
// Per slot, if every stored item has the same policy score (LCBFU: all f = 0, the never-
// accessed bulk; LRU / LFU: equal columns; FIFO: always) its keys are S<<35 | id<<3 | j, a run
// of <= 5 consecutive values: one bin / range test for the whole slot instead of 5 key builds.
// The output claims are aggregated per lane (20-bit masks) and per warp (one scan, one atomic
// per list and warp iteration) instead of a warp ballot + atomic per item.
__device__ __forceinline__ unsigned long long warp_excl_scan_u64(unsigned long long x, int lane,
                                                                 unsigned long long* total) {
    unsigned long long v = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, v, o);
        if (lane >= o) v += y;
    }
    *total = __shfl_sync(0xFFFFFFFFu, v, 31);
    return v - x;
}
// one atomic per warp: this lane's first output index of `cnt` items
__device__ __forceinline__ unsigned long long warp_reserve(unsigned long long* counter, uint32_t cnt, int lane) {
    unsigned long long tot = 0;
    const unsigned long long ex = warp_excl_scan_u64(cnt, lane, &tot);
    unsigned long long base = 0;
    if (lane == 0 && tot) base = atomicAdd(counter, tot);
    base = __shfl_sync(0xFFFFFFFFu, base, 0);
    return base + ex;
}

template <int POLICY>
__device__ __forceinline__ uint32_t sat_score(uint32_t col, int kvj, uint32_t limj) {
    if constexpr (POLICY == CACHE_POLICY_LCBFU) return col > limj ? 0x1FFFFFFFu : col * (uint32_t)kvj;
    else if constexpr (POLICY == CACHE_POLICY_FIFO) return 0u;
    else return col > 0x1FFFFFFFu ? 0x1FFFFFFFu : col;
}
__device__ __forceinline__ unsigned long long mk_key(uint32_t sc, uint32_t id, int j) {
    return ((unsigned long long)sc << 35) | ((unsigned long long)id << 3) | (unsigned long long)j;
}

template <int POLICY>
__device__ __forceinline__ void sweep_items_v4(const SelArgs& a, const int (&kv)[CACHE_MAX_K],
                                               const uint32_t (&lim)[CACHE_MAX_K], int mode, const SelLevel& L,
                                               int64_t e4, const uint32_t (&pm)[4], const uint32_t (&pid)[4],
                                               const uint32_t (&c)[20], unsigned* sh, DigitRun& run,
                                               unsigned long long& kmin, int lane) {
    uint32_t evm = 0u, inm = 0u;   // bit 5q + j: item j of slot q is evicted / in the range
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint32_t m = pm[q] & 31u, id = pid[q];
        if (!m) continue;
        bool uni;
        uint32_t S = 0u;
        if constexpr (POLICY == CACHE_POLICY_FIFO) uni = true;
        else if constexpr (POLICY == CACHE_POLICY_LCBFU)
            uni = (c[5 * q] | c[5 * q + 1] | c[5 * q + 2] | c[5 * q + 3] | c[5 * q + 4]) == 0u;
        else {
            uni = c[5 * q] == c[5 * q + 1] && c[5 * q] == c[5 * q + 2] && c[5 * q] == c[5 * q + 3] &&
                  c[5 * q] == c[5 * q + 4];
            S = sat_score<POLICY>(c[5 * q], 0, 0u);
        }
        const unsigned long long k0 = mk_key(S, id, __ffs(m) - 1), k1 = mk_key(S, id, 31 - __clz(m));
        bool done = false;
        bool wdone = !(mode == kSweepL0 && L.compact);   // single-sweep window bits (keys < L.T)
        if (uni) {
            if (mode == kSweepL0) {
                const uint32_t b = sel_bin0(k0);
                if (b == sel_bin0(k1)) {
                    run.add_n(sh, b, (unsigned)__popc(m));
                    kmin = k0 < kmin ? k0 : kmin;
                    done = true;
                }
                if (!wdone) {
                    if (k1 < L.T) { inm |= m << (5 * q); wdone = true; }
                    else if (k0 >= L.T) wdone = true;
                }
            } else if (mode == kSweepFinal) {
                if (k1 <= L.T) { evm |= m << (5 * q); done = true; }
                else if (k0 > L.T) done = true;
            } else {
                if (k1 < L.lo) { evm |= m << (5 * q); done = true; }
                else if (k0 >= L.lo && ((k0 - L.lo) >> L.w) != 0ull) done = true;   // above the range
                else if (k0 >= L.lo && ((k1 - L.lo) >> L.w) == 0ull &&
                         ((k0 - L.lo) >> L.shift) == ((k1 - L.lo) >> L.shift)) {
                    inm |= m << (5 * q);
                    const uint32_t d = (uint32_t)((k0 - L.lo) >> L.shift);
                    run.add_n(sh, d, (unsigned)__popc(m));
                    done = true;
                }
            }
        }
        if (!done || !wdone) {
#pragma unroll
            for (int j = 0; j < 5; ++j) {
                if (!((m >> j) & 1u)) continue;
                const unsigned long long key = mk_key(sat_score<POLICY>(c[5 * q + j], kv[j], lim[j]), id, j);
                if (mode == kSweepL0) {
                    if (!done) {
                        run.add(sh, sel_bin0(key));
                        kmin = key < kmin ? key : kmin;
                    }
                    if (!wdone && key < L.T) inm |= 1u << (5 * q + j);
                } else if (mode == kSweepFinal) {
                    if (key <= L.T) evm |= 1u << (5 * q + j);
                } else if (key < L.lo) {
                    evm |= 1u << (5 * q + j);
                } else if (((key - L.lo) >> L.w) == 0ull) {
                    inm |= 1u << (5 * q + j);
                    run.add(sh, (uint32_t)((key - L.lo) >> L.shift));
                }
            }
        }
    }
    if (mode == kSweepL0) {
        if (L.compact && __any_sync(0xFFFFFFFFu, inm != 0u)) {   // warp-uniform: the window's (key, slot) pairs
            unsigned long long wpos = warp_reserve(&a.out->cnt_w, (uint32_t)__popc(inm), lane);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t inq = (inm >> (5 * q)) & 31u;
                if (!inq) continue;
#pragma unroll
                for (int j = 0; j < 5; ++j) {
                    if (!((inq >> j) & 1u)) continue;
                    if (wpos < a.cand_cap) {
                        a.cand_key[wpos] = mk_key(sat_score<POLICY>(c[5 * q + j], kv[j], lim[j]), pid[q], j);
                        a.cand_slot[wpos] = (uint32_t)(e4 + q);
                    }
                    ++wpos;
                }
            }
        }
        return;
    }
    // outputs: evicted keys (one warp reservation), candidates, presence / counters / dirty
    unsigned long long pos = warp_reserve(&a.out->cnt[0], (uint32_t)__popc(evm), lane);
    unsigned long long cpos = 0;
    if (mode == kSweepLevel && L.compact) cpos = warp_reserve(&a.out->cnt[3], (uint32_t)__popc(inm), lane);
    uint32_t ndirty = 0;
    BitRun evr;
    // dirty slots: the lane's 4 slots lie in one bitmap word, shared by lanes 8k .. 8k+7 (one
    // atomic per word after a 3-step OR); dirty ids / world: a word run per lane, then OR'ed
    // across neighbouring lanes (consecutive ids)
    uint32_t dsm = 0u;
    WordRun dir;
    // LCBFU / LFU: the lane's 20 counters are in c[] -- written back with 5 vector stores, the
    // evicted ones zeroed (no query runs during an eviction)
    constexpr bool kVecF = POLICY == CACHE_POLICY_LCBFU || POLICY == CACHE_POLICY_LFU;
    if constexpr (kVecF) {
        if (evm) {
            uint4* fp = reinterpret_cast<uint4*>(a.fcnt + e4 * 5);
#pragma unroll
            for (int v = 0; v < 5; ++v) {
                if (!((evm >> (4 * v)) & 15u)) continue;
                uint4 o;
                o.x = (evm >> (4 * v)) & 1u ? 0u : c[4 * v];
                o.y = (evm >> (4 * v + 1)) & 1u ? 0u : c[4 * v + 1];
                o.z = (evm >> (4 * v + 2)) & 1u ? 0u : c[4 * v + 2];
                o.w = (evm >> (4 * v + 3)) & 1u ? 0u : c[4 * v + 3];
                fp[v] = o;
            }
        }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint32_t m = pm[q] & 31u, id = pid[q];
        const uint32_t evq = (evm >> (5 * q)) & 31u, inq = (inm >> (5 * q)) & 31u;
        if (!(evq | (L.compact ? inq : 0u))) continue;
        const int64_t e = e4 + q;
#pragma unroll
        for (int j = 0; j < 5; ++j) {
            if (!(((evq | inq) >> j) & 1u)) continue;
            const unsigned long long key = mk_key(sat_score<POLICY>(c[5 * q + j], kv[j], lim[j]), id, j);
            if ((evq >> j) & 1u) {
                if (pos < a.ev_cap) a.ev_key[pos] = key;
                ++pos;
                evr.add(a, L, key);
                if constexpr (!kVecF) a.fcnt[e * 5 + j] = 0u;
            } else if (mode == kSweepLevel && L.compact) {
                if (cpos < a.cand_cap) { a.cand_key[cpos] = key; a.cand_slot[cpos] = (uint32_t)e; }
                ++cpos;
            }
        }
        if (evq) {
            const uint32_t keep = m & ~evq;
            a.present[e] = keep | (pm[q] & ~31u);
            if (!keep) {
                a.inv_e[e] = __int_as_float(0x7FC00000);
                dsm |= 1u << (e & 31);
                dir.add(a.did_bits, id / (uint32_t)a.world);   // ids of this rank: id % world == rank
                ++ndirty;
            }
        }
    }
    // freed pool slots: the lane's 20 latent-slot entries by 5 independent vector loads (a
    // scalar load per evicted item behind the previous item's atomic was a chain of up to 20
    // round trips: the C2 eviction's slowest warps, NV_SEL_TRACE)
    if (a.pool_bits && evm) {
        int4 lv[5];
        const int4* lp = reinterpret_cast<const int4*>(a.lslot + e4 * 5);
#pragma unroll
        for (int v = 0; v < 5; ++v) lv[v] = __ldg(lp + v);
        WordRun plr;
#pragma unroll
        for (int v = 0; v < 5; ++v) {
            const int32_t x[4] = {lv[v].x, lv[v].y, lv[v].z, lv[v].w};
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (((evm >> (4 * v + k)) & 1u) && x[k] >= 0) plr.add(a.pool_bits, (uint32_t)x[k]);
        }
        if (plr.m) atomicOr(a.pool_bits + plr.w, plr.m);
    }
    {
        uint32_t x = dsm;
        x |= __shfl_xor_sync(0xFFFFFFFFu, x, 1);
        x |= __shfl_xor_sync(0xFFFFFFFFu, x, 2);
        x |= __shfl_xor_sync(0xFFFFFFFFu, x, 4);
        if ((lane & 7) == 0 && x) atomicOr(a.dslot_bits + (e4 >> 5), x);
    }
    dir.warp_flush(a.did_bits, lane);
    evr.flush(a);
    unsigned long long dt = 0;
    (void)warp_excl_scan_u64(ndirty, lane, &dt);
    if (lane == 0 && dt) atomicAdd(&a.out->cnt[1], dt);
}

// ---- TMA bulk staging of the slot columns (the |K| = 5 full sweeps): one thread streams
// 2,048-slot tiles (present 8 KB, ids 8 KB, policy column 40 KB) into a 3-stage shared-memory
// ring with cp.async.bulk; the 16 warps read their 4 slots per lane from shared memory.  The
// bytes in flight no longer depend on registers: the register-fed version (7 x 16-B loads per
// lane, 2 CTAs / SM) reached 2.98 TB/s = 0.45 of the copy peak, latency-bound (ncu). ----
#ifndef NV_SEL_STAGED
#define NV_SEL_STAGED 0   // 1: the TMA-staged sweep (measured slower, kept for the record)
#endif
constexpr bool kSelStaged = NV_SEL_STAGED != 0;
constexpr int kTile = 2048, kStages = 3;
constexpr int kStageBytes = kTile * 4 * 7;   // present + ids + 5 columns
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void bar_wait(uint32_t bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done) : "r"(bar), "r"(parity) : "memory");
    }
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}

template <int POLICY>
__device__ __forceinline__ const uint32_t* policy_col(const SelArgs& a) {
    if constexpr (POLICY == CACHE_POLICY_LRU) return a.lastacc;
    else return a.fcnt;
}

// Candidate i (key, slot): histogram (level) or apply (final, key <= T).
template <int POLICY, int GRAN>
__device__ __forceinline__ void sel_cand(const SelArgs& a, const KMap& km, int mode, const SelLevel& L, int64_t i,
                                         bool valid, unsigned* sh, DigitRun& run, int lane) {
    const int nk = km.num_k;
    const unsigned long long key = valid ? a.cand_key[i] : 0ull;
    const int64_t e = valid ? (int64_t)a.cand_slot[i] : 0;
    if (mode == kSweepLevel) {
        if (valid && key >= L.lo && ((key - L.lo) >> L.w) == 0ull) run.add(sh, (unsigned)((key - L.lo) >> L.shift));
        return;
    }
    const bool ev = valid && key <= L.T;
    const unsigned long long at = warp_claim(&a.out->cnt[0], ev, lane);
    if constexpr (GRAN == CACHE_EVICT_ENTRY) {
        (void)warp_claim(&a.out->cnt[1], ev, lane);
        if (ev) {
            const uint32_t m = a.present[e];
            atomicAdd(&a.out->cnt[2], (unsigned long long)__popc(m));
            for (int j = 0; j < nk; ++j) {
                if ((m >> j) & 1u) mark_pool(a, a.lslot[e * nk + j]);
                a.fcnt[e * nk + j] = 0u;
            }
            a.present[e] = 0u;
            a.inv_e[e] = __int_as_float(0x7FC00000);
            mark_dirty(a, e, (uint32_t)(key & 0xFFFFFFFFull));
            if (at < a.ev_cap) a.ev_key[at] = key;
            ev_mark(a, L, key);
        }
    } else {
        bool dirty = false;
        if (ev) {
            const int j = (int)(key & 7ull);
            const uint32_t bit = 1u << j;
            if (at < a.ev_cap) a.ev_key[at] = key;
            ev_mark(a, L, key);
            mark_pool(a, a.lslot[e * nk + j]);
            a.fcnt[e * nk + j] = 0u;
            const uint32_t old = atomicAnd(a.present + e, ~bit);   // the entry's last bit -> dirty
            dirty = (old & ~bit) == 0u;
            if (dirty) {
                a.inv_e[e] = __int_as_float(0x7FC00000);
                mark_dirty(a, e, (uint32_t)((key >> 3) & 0xFFFFFFFFull));
            }
        }
        (void)warp_claim(&a.out->cnt[1], dirty, lane);
    }
}

// The final apply over the candidates, item mode (the single-sweep window's whole apply: ~n
// candidates), warp-aggregated: the candidates of one slot sit in consecutive buffer positions
// (a lane compacts a slot's items together), so each run of lanes with the same slot clears its
// presence bits with ONE atomicAnd (the run that clears the slot's last bit makes it dirty), and
// the evicted-key, pool-slot, dirty-slot and dirty-id bitmaps take one atomic per word.  (Per
// candidate, the atomics on shared words serialised: 41 us for 619K candidates, NV_SEL_TRACE.)
// ev_list: also write the unsorted evicted-key list (only when the key bitmap may not cover every
// evicted key: one counter claim per warp and iteration -- one address, so ~20K serialised
// atomics over a 619K-item apply); the counts go to *nev / *ndirty (per lane, summed by the caller).
__device__ __forceinline__ void cand_apply_item(const SelArgs& a, int nk, const SelLevel& L, int64_t i, bool valid,
                                                int lane, bool ev_list, uint32_t& nev, uint32_t& ndirty) {
    const unsigned long long key = valid ? __ldcg(a.cand_key + i) : ~0ull;
    const uint32_t e = valid ? __ldcg(a.cand_slot + i) : 0xFFFFFFFFu;
    const bool ev = valid && key <= L.T;
    const int j = (int)(key & 7ull);
    if (ev_list) {   // grid-uniform
        const unsigned long long at = warp_claim(&a.out->cnt[0], ev, lane);
        if (ev && at < a.ev_cap) a.ev_key[at] = key;
    } else {
        nev += ev ? 1u : 0u;
    }
    if (L.ev_lim) {   // grid-uniform
        WordRun r;
        if (ev) {
            const unsigned long long d = key - L.kb;
            if (d >= L.ev_lim) atomicExch(&a.out->ev_over, 1u);   // overflow: sort on the host side
            else r.add(a.ev_bits, (uint32_t)d);
        }
        r.warp_flush(a.ev_bits, lane);
    }
    if (a.pool_bits) {   // grid-uniform
        WordRun r;
        if (ev) {
            const int32_t ps = __ldg(a.lslot + (int64_t)e * nk + j);
            if (ps >= 0) r.add(a.pool_bits, (uint32_t)ps);
        }
        r.warp_flush(a.pool_bits, lane);
    }
    if (ev) a.fcnt[(int64_t)e * nk + j] = 0u;
    // presence: a segmented OR over runs of lanes with the same slot (strictly contiguous runs:
    // a slot repeated further on forms its own run with disjoint bits)
    const uint32_t me = ev ? e : 0xFFFFFFFFu;
    const uint32_t prev = __shfl_up_sync(0xFFFFFFFFu, me, 1);
    const bool start = lane == 0 || prev != me;
    const unsigned starts = __ballot_sync(0xFFFFFFFFu, start);
    const unsigned after = starts & ~((2u << lane) - 1u);   // (2u << 31) == 0: no later run
    const int nh = after ? __ffs(after) - 1 : 32;           // first lane of the next run
    uint32_t acc = ev ? (1u << j) : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t ob = __shfl_down_sync(0xFFFFFFFFu, acc, o);
        if (lane + o < nh) acc |= ob;
    }
    bool dirty = false;
    if (ev && start) {
        const uint32_t old = atomicAnd(a.present + e, ~acc);
        dirty = (old & ~acc) == 0u;
        if (dirty) a.inv_e[e] = __int_as_float(0x7FC00000);
    }
    WordRun ds, di;
    if (dirty) {
        ds.add(a.dslot_bits, e);
        di.add(a.did_bits, (uint32_t)((key >> 3) & 0xFFFFFFFFull) / (uint32_t)a.world);
    }
    ds.warp_flush(a.dslot_bits, lane);
    di.warp_flush(a.did_bits, lane);
    ndirty += dirty ? 1u : 0u;
}

// Ordered compaction of the bitmaps into ascending lists (dirty slots, dirty ids, freed pool
// slots, evicted keys): per CTA a contiguous word range; CTA totals are exchanged through global
// memory across one grid barrier.  Inside a CTA the range goes in rounds of kSelThreads words
// (one per thread, a block scan of their popcounts), and each warp emits its words' bits one
// word at a time with lane = bit, so every output store is coalesced.  (The first version gave
// each thread a contiguous sub-range and wrote its bits one by one: the dirty bitmaps are dense
// in the oldest slots, so the first CTAs issued ~200 scattered 8-B stores per thread -- a 60-us
// tail at 12.5M entries, NV_SEL_TRACE.)
struct BitJob {
    const uint32_t* bits;
    int64_t words;
    unsigned long long* out;
    unsigned long long mul, add;   // value of bit i = i * mul + add
    unsigned long long* out2;      // optional second list: value & mask2
    unsigned long long mask2;
};

__device__ __forceinline__ uint32_t block_excl_scan_u32(uint32_t x, uint32_t* total) {
    __shared__ uint32_t s_ws[kSelThreads / 32];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    uint32_t v = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, v, o);
        if (lane >= o) v += y;
    }
    if (lane == 31) s_ws[w] = v;
    __syncthreads();
    uint32_t off = 0, tot = 0;
    for (int i = 0; i < kSelThreads / 32; ++i) {
        off += i < w ? s_ws[i] : 0u;
        tot += s_ws[i];
    }
    __syncthreads();
    *total = tot;
    return off + v - x;
}

template <int NJ>
__device__ void compact_bitmaps(const BitJob (&jobs)[NJ], uint32_t* part, cg::grid_group& grid, int& ts) {
    // Chunks of kSelThreads words (one per thread) of the jobs' bitmaps, concatenated and dealt
    // round-robin to the CTAs (flat chunk f -> CTA f % grid): the dense runs of the dirty bitmaps
    // (the oldest slots) land on many CTAs (contiguous per-CTA ranges left 3 CTAs emitting 125K
    // values each: a 25-us tail per list, NV_SEL_TRACE).  part[f] = chunk totals; after the grid
    // barrier every CTA scans ALL the totals (a few per thread) for the bases of its own chunks,
    // so no chunk waits on another; loads are batched kCB chunks at a time.
    constexpr int kCB = 8, kOwnMax = 256;
    __shared__ uint32_t s_red[kCB][kSelThreads / 32];
    __shared__ uint32_t s_base[kOwnMax];    // global prefix of own chunk k (all jobs)
    __shared__ uint32_t s_jpre[NJ];         // global prefix at each job's first chunk
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t G = gridDim.x;
    int64_t nch[NJ], off[NJ];
    int64_t total = 0;
#pragma unroll
    for (int q = 0; q < NJ; ++q) {
        nch[q] = jobs[q].bits ? (jobs[q].words + kSelThreads - 1) / kSelThreads : 0;
        off[q] = total;
        total += nch[q];
    }
    auto job_of = [&](int64_t f) {
        int q = 0;
#pragma unroll
        for (int k = 1; k < NJ; ++k)
            if (f >= off[k] && nch[k]) q = k;
        return q;
    };
    auto word_of = [&](int64_t f) -> uint32_t {   // this thread's word of flat chunk f
        if (f >= total) return 0u;
        const int q = job_of(f);
        const int64_t w = (f - off[q]) * kSelThreads + threadIdx.x;
        uint32_t m = 0u;
#pragma unroll
        for (int k = 0; k < NJ; ++k)
            if (k == q && w < jobs[k].words) m = __ldcg(jobs[k].bits + w);
        return m;
    };
    // part 1: the totals of this CTA's chunks
    for (int64_t f0 = blockIdx.x; f0 < total; f0 += kCB * G) {   // CTA-uniform
        uint32_t cnt[kCB];
#pragma unroll
        for (int k = 0; k < kCB; ++k) cnt[k] = word_of(f0 + k * G);
#pragma unroll
        for (int k = 0; k < kCB; ++k) {
            uint32_t v = __popc(cnt[k]);
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
            if (lane == 0) s_red[k][warp] = v;
        }
        __syncthreads();
        if (threadIdx.x < kCB && f0 + threadIdx.x * G < total) {
            uint32_t t = 0;
#pragma unroll
            for (int i = 0; i < kSelThreads / 32; ++i) t += s_red[threadIdx.x][i];
            part[f0 + threadIdx.x * G] = t;
        }
        __syncthreads();
    }
    sel_stamp(ts);
    grid.sync();
    sel_stamp(ts);
    // every CTA: exclusive scan of all totals (thread t: a contiguous run of them)
    {
        const int64_t per = (total + kSelThreads - 1) / kSelThreads;
        const int64_t i0 = min(total, (int64_t)threadIdx.x * per), i1 = min(total, i0 + per);
        uint32_t sum = 0;
        for (int64_t i = i0; i < i1; ++i) sum += __ldcg(part + i);
        uint32_t tot = 0;
        uint32_t run = block_excl_scan_u32(sum, &tot);
        for (int64_t i = i0; i < i1; ++i) {
#pragma unroll
            for (int q = 0; q < NJ; ++q)
                if (nch[q] && i == off[q]) s_jpre[q] = run;
            if (i >= blockIdx.x && (i - blockIdx.x) % G == 0 && (i - blockIdx.x) / G < kOwnMax)
                s_base[(i - blockIdx.x) / G] = run;
            run += __ldcg(part + i);
        }
        __syncthreads();
    }
    // part 2: emission, kCB own chunks per batch (their words loaded together)
    for (int64_t f0 = blockIdx.x, k0 = 0; f0 < total; f0 += kCB * G, k0 += kCB) {   // CTA-uniform
        uint32_t mw[kCB];
#pragma unroll
        for (int k = 0; k < kCB; ++k) mw[k] = word_of(f0 + k * G);
#pragma unroll
        for (int k = 0; k < kCB; ++k) {
            const int64_t f = f0 + k * G;
            if (f >= total) break;   // CTA-uniform
            const int q = job_of(f);
            const int64_t c = f - off[q];
            uint32_t base;
            if (k0 + k < kOwnMax) {
                base = s_base[k0 + k] - s_jpre[q];
            } else {   // more own chunks than the table holds: sum the job's earlier totals
                uint32_t v = 0;
                for (int64_t i = off[q] + threadIdx.x; i < f; i += kSelThreads) v += __ldcg(part + i);
                (void)block_excl_scan_u32(v, &base);
            }
            const uint32_t m = mw[k];
            uint32_t tot = 0;
            const uint32_t offw = block_excl_scan_u32((uint32_t)__popc(m), &tot);
            unsigned long long* out = nullptr;
            unsigned long long* out2 = nullptr;
            unsigned long long mul = 0, add = 0, mask2 = 0;
#pragma unroll
            for (int kk = 0; kk < NJ; ++kk)
                if (kk == q) { out = jobs[kk].out; out2 = jobs[kk].out2; mul = jobs[kk].mul; add = jobs[kk].add; mask2 = jobs[kk].mask2; }
            unsigned nz = __ballot_sync(0xFFFFFFFFu, m != 0u);
            while (nz) {   // warp-uniform: one word at a time, lane = bit (coalesced stores)
                const int j = __ffs(nz) - 1;
                nz &= nz - 1u;
                const uint32_t mj = __shfl_sync(0xFFFFFFFFu, m, j);
                const uint32_t oj = __shfl_sync(0xFFFFFFFFu, offw, j);
                if ((mj >> lane) & 1u) {
                    const unsigned long long pos = (unsigned long long)base + oj + __popc(mj & ((1u << lane) - 1u));
                    const int64_t bit = (c * kSelThreads + warp * 32 + j) * 32 + lane;
                    const unsigned long long v = (unsigned long long)bit * mul + add;
                    if (out2) out2[pos] = v & mask2;
                    out[pos] = v;
                }
            }
        }
    }
    sel_stamp(ts);
}

// NK5: |K| = 5 (the paper's): every lane loads 4 consecutive slots with 16-byte loads (presence,
// ids, 5 x the policy column = 20 u32) -- 7 independent loads in flight per thread instead of a
// dependent present -> id -> counter chain per slot (ncu: the first version moved 704 MB in
// 789 us, 0.9 TB/s, stalled on those chains and on the grid barrier behind them).
template <int POLICY, int GRAN, bool NK5>
__global__ void __launch_bounds__(kSelThreads, (NK5 && kSelStaged) ? 1 : ((kSelCpAsync || kSelPrefetch) ? 3 : 2))
    k_evict_select(SelArgs a, KMap km) {
    __shared__ unsigned sh[kSelBins];
    __shared__ __align__(8) unsigned long long s_bar[2 * kStages];   // full[s], empty[s]
    extern __shared__ __align__(128) unsigned char s_stage[];        // NK5: TMA stages / cp.async ring
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int kv[CACHE_MAX_K];
#pragma unroll
    for (int j = 0; j < CACHE_MAX_K; ++j) kv[j] = km.kv[j];
    // the sweeps interleave 128-slot groups (one warp iteration of the vector path) over all
    // warps of the grid: the evictions concentrate in the oldest slots, and contiguous
    // per-CTA slices left a few CTAs with all the output claims behind a grid barrier (ncu:
    // 41% of the warps' time in stall_barrier).  The arrays are padded to 256 slots and slots
    // >= hwm are never live.
    const int64_t n_pad = (a.n_slots + 127) & ~(int64_t)127;
    const int nk = NK5 ? 5 : km.num_k;
    uint32_t lim[CACHE_MAX_K];   // LCBFU saturation: f > lim[j] <=> f * K_j > 2^29 - 1 (R11)
#pragma unroll
    for (int j = 0; j < CACHE_MAX_K; ++j) lim[j] = kv[j] > 0 ? 0x1FFFFFFFu / (uint32_t)kv[j] : 0xFFFFFFFFu;
    auto clear_sh = [&]() {
        for (int i = threadIdx.x; i < kSelBins; i += kSelThreads) sh[i] = 0u;
        __syncthreads();
    };
    auto flush_sh = [&](uint32_t* gh) {
        __syncthreads();
        for (int i = threadIdx.x; i < kSelBins; i += kSelThreads)
            if (sh[i]) atomicAdd(gh + i, sh[i]);
    };
    if constexpr (NK5 && kSelStaged) {
        if (threadIdx.x == 0) {
            for (int st = 0; st < kStages; ++st) {
                bar_init(su32(&s_bar[st]), 1);                         // full: the producer's expect_tx
                bar_init(su32(&s_bar[kStages + st]), kSelThreads / 32); // empty: one arrive per warp
            }
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
    }
    uint32_t uses = 0;   // tiles this CTA has staged so far (all sweeps): stage = u % kStages
    int sweep_no = 0;    // full sweeps so far (each has its own claim counter)
    auto full_sweep = [&](int mode, const SelLevel& L, unsigned long long& kmin) {
        DigitRun run;
        const uint32_t* colp = policy_col<POLICY>(a);
        if constexpr (NK5 && kSelStaged) {
            const int64_t ntiles = (n_pad + kTile - 1) / kTile;
            const int64_t mine = ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
            // tile k of this CTA = global tile blockIdx.x + k * gridDim.x (interleaved)
            auto issue = [&](int64_t k) {
                const uint32_t u = uses + (uint32_t)k, st = u % kStages;
                if (u >= (uint32_t)kStages) bar_wait(su32(&s_bar[kStages + st]), ((u / kStages) - 1) & 1);
                const int64_t t0 = (blockIdx.x + k * gridDim.x) * (int64_t)kTile;
                const uint32_t cnt = (uint32_t)min((int64_t)kTile, n_pad - t0);   // a multiple of 128
                const uint32_t full = su32(&s_bar[st]);
                unsigned char* base = s_stage + (size_t)st * kStageBytes;
                const uint32_t colb = POLICY != CACHE_POLICY_FIFO ? cnt * 20u : 0u;
                bar_expect_tx(full, cnt * 8u + colb);
                bulk_g2s(su32(base), a.present + t0, cnt * 4u, full);
                bulk_g2s(su32(base + kTile * 4), a.ids + t0, cnt * 4u, full);
                if (colb) bulk_g2s(su32(base + kTile * 8), colp + t0 * 5, colb, full);
            };
            if (threadIdx.x == 0) {
                asm volatile("fence.proxy.async.global;" ::: "memory");   // earlier sweeps' stores -> TMA reads
                for (int64_t k = 0; k < (mine < kStages ? mine : (int64_t)kStages); ++k) issue(k);
            }
            for (int64_t k = 0; k < mine; ++k) {
                const uint32_t u = uses + (uint32_t)k, st = u % kStages;
                bar_wait(su32(&s_bar[st]), (u / kStages) & 1);
                const int64_t t0 = (blockIdx.x + k * gridDim.x) * (int64_t)kTile;
                const int64_t e4 = t0 + 4 * threadIdx.x;   // 4 slots of this lane
                const bool in = e4 < n_pad;
                const unsigned char* base = s_stage + (size_t)st * kStageBytes;
                const uint4 P = in ? reinterpret_cast<const uint4*>(base)[threadIdx.x] : make_uint4(0, 0, 0, 0);
                const uint4 I = reinterpret_cast<const uint4*>(base + kTile * 4)[threadIdx.x];
                uint32_t c[20];
                if constexpr (POLICY != CACHE_POLICY_FIFO) {
                    const uint4* cp = reinterpret_cast<const uint4*>(base + kTile * 8) + 5 * threadIdx.x;
#pragma unroll
                    for (int v = 0; v < 5; ++v) {
                        const uint4 w = cp[v];
                        c[4 * v] = w.x; c[4 * v + 1] = w.y; c[4 * v + 2] = w.z; c[4 * v + 3] = w.w;
                    }
                } else {
#pragma unroll
                    for (int v = 0; v < 20; ++v) c[v] = 0u;
                }
                __syncwarp();
                if (lane == 0) bar_arrive(su32(&s_bar[kStages + st]));   // this warp is done with the stage
                if (threadIdx.x == 0 && k + kStages < mine) issue(k + kStages);
                const uint32_t pm[4] = {P.x, P.y, P.z, P.w}, pid[4] = {I.x, I.y, I.z, I.w};
                if constexpr (GRAN == CACHE_EVICT_ITEM) {
                    sweep_items_v4<POLICY>(a, kv, lim, mode, L, e4, pm, pid, c, sh, run, kmin, lane);
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        uint32_t col[CACHE_MAX_K];
#pragma unroll
                        for (int j = 0; j < CACHE_MAX_K; ++j) col[j] = j < 5 ? c[5 * q + j] : 0u;
                        sel_slot<POLICY, GRAN>(a, 5, kv, mode, L, e4 + q, pm[q], pid[q], col, sh, run, kmin, lane);
                    }
                }
            }
            uses += (uint32_t)mine;
        } else if constexpr (NK5 && kSelCpAsync) {
            // per-lane cp.async ring: each lane copies its own 112 B per group (present, ids and
            // the 5-word column of 4 consecutive slots) straight into shared memory, two groups
            // ahead of the one it processes -- loads in flight without holding registers
            // (the register-fed loop keeps one group in flight per lane, 0.44 of the copy peak)
            const int64_t gstride = (int64_t)gridDim.x * 4 * kSelThreads;
            const int64_t gfirst = ((int64_t)blockIdx.x * (kSelThreads / 32) + warp) * 128;
            uint4* ring = reinterpret_cast<uint4*>(s_stage);
            auto slot_of = [&](int st) { return ring + ((size_t)st * kSelThreads + threadIdx.x) * 7; };
            auto issue = [&](int64_t g0, int st) {
                if (g0 < n_pad) {
                    const int64_t e4 = g0 + 4 * lane;
                    const uint32_t d = su32(slot_of(st));
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(a.present + e4) : "memory");
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d + 16), "l"(a.ids + e4) : "memory");
                    if constexpr (POLICY != CACHE_POLICY_FIFO) {
#pragma unroll
                        for (int v = 0; v < 5; ++v)
                            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d + 32 + 16 * v),
                                         "l"(colp + e4 * 5 + 4 * v) : "memory");
                    }
                }
                asm volatile("cp.async.commit_group;" ::: "memory");   // (possibly empty) one group per iteration
            };
            issue(gfirst, 0);
            issue(gfirst + gstride, 1);
            int st = 0;
            for (int64_t g0 = gfirst; g0 < n_pad; g0 += gstride) {
                issue(g0 + 2 * gstride, (st + 2) % kCpStages);
                asm volatile("cp.async.wait_group 2;" ::: "memory");   // this iteration's group landed
                const uint4* sl = slot_of(st);
                const uint4 P = sl[0], I = sl[1];
                uint32_t c[20];
                if constexpr (POLICY != CACHE_POLICY_FIFO) {
#pragma unroll
                    for (int v = 0; v < 5; ++v) {
                        const uint4 w = sl[2 + v];
                        c[4 * v] = w.x; c[4 * v + 1] = w.y; c[4 * v + 2] = w.z; c[4 * v + 3] = w.w;
                    }
                } else {
#pragma unroll
                    for (int v = 0; v < 20; ++v) c[v] = 0u;
                }
                st = (st + 1) % kCpStages;
                const int64_t e4 = g0 + 4 * lane;
                const uint32_t pm[4] = {P.x, P.y, P.z, P.w}, pid[4] = {I.x, I.y, I.z, I.w};
                if constexpr (GRAN == CACHE_EVICT_ITEM) {
                    sweep_items_v4<POLICY>(a, kv, lim, mode, L, e4, pm, pid, c, sh, run, kmin, lane);
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        uint32_t col[CACHE_MAX_K];
#pragma unroll
                        for (int j = 0; j < CACHE_MAX_K; ++j) col[j] = j < 5 ? c[5 * q + j] : 0u;
                        sel_slot<POLICY, GRAN>(a, 5, kv, mode, L, e4 + q, pm[q], pid[q], col, sh, run, kmin, lane);
                    }
                }
            }
            asm volatile("cp.async.wait_group 0;" ::: "memory");   // drain the empty tail groups
        } else if constexpr (NK5) {
            // register-fed: 7 independent 16-B loads per lane (present, ids, 5 x the column of
            // 4 consecutive slots); 128-slot groups interleaved over all warps of the grid
            const int64_t gstride = (int64_t)gridDim.x * 4 * kSelThreads;
            const int64_t gfirst = ((int64_t)blockIdx.x * (kSelThreads / 32) + warp) * 128;
            // kSelPrefetch: the next group's seven loads are issued before this group is
            // processed (3 CTAs of 256 threads per SM at <= 85 registers), so a lane keeps one
            // group in flight while it works instead of alternating load and work
            uint4 nP = make_uint4(0, 0, 0, 0), nI = nP, nC[5] = {nP, nP, nP, nP, nP};
            auto load = [&](int64_t g, uint4& P_, uint4& I_, uint4 (&C_)[5]) {
                const int64_t e = g + 4 * lane;
                P_ = __ldcg(reinterpret_cast<const uint4*>(a.present + e));
                I_ = __ldcg(reinterpret_cast<const uint4*>(a.ids + e));
                if constexpr (POLICY != CACHE_POLICY_FIFO) {
                    if constexpr (kSelColT) {
                        // the warp's 2,560-B column block in five fully coalesced 512-B loads,
                        // redistributed through shared memory to the lanes' own 4 slots (the
                        // per-lane 80-B reads touched 20 lines per load instruction)
                        const uint4* cp = reinterpret_cast<const uint4*>(colp + g * 5);
                        uint4* tr = reinterpret_cast<uint4*>(s_stage) + warp * 160;   // dynamic smem
#pragma unroll
                        for (int v = 0; v < 5; ++v) C_[v] = __ldcg(cp + lane + 32 * v);
#pragma unroll
                        for (int v = 0; v < 5; ++v) tr[lane + 32 * v] = C_[v];
                        __syncwarp();
#pragma unroll
                        for (int v = 0; v < 5; ++v) C_[v] = tr[5 * lane + v];
                        __syncwarp();
                    } else {
                        const uint4* cp = reinterpret_cast<const uint4*>(colp + e * 5);
#pragma unroll
                        for (int v = 0; v < 5; ++v) C_[v] = __ldcg(cp + v);
                    }
                }
            };
            if (kSelPrefetch && gfirst < n_pad) load(gfirst, nP, nI, nC);
            // NV_SEL_DYN_PCT > 0 (single-cache launch): the last DYN_PCT% of the groups are claimed
            // (2 per atomic) by whichever warps finish their static share first -- the static
            // interleave keeps the bulk's access pattern, the claimed tail absorbs the CTAs that
            // run 20-25% slower than the median (NV_SEL_TRACE)
            const int64_t ngroups = n_pad / 128, twarps = (int64_t)gridDim.x * (kSelThreads / 32);
            int64_t dyn_from = ngroups;   // groups >= dyn_from are claimed
            if (kSelDynPct > 0 && a.phase == kPhaseAll && !kSelPrefetch && sweep_no < 16)   // a counter per sweep
                dyn_from = (ngroups / twarps) * (100 - kSelDynPct) / 100 * twarps;
            unsigned long long* gctr = &a.out->gnext[(sweep_no++) & 15];
            bool in_dyn = gfirst >= dyn_from * 128;
            int dleft = 0;
            int64_t dnext = 0, g0 = gfirst;
            for (;;) {
                if (in_dyn) {   // warp-uniform
                    if (dyn_from >= ngroups) break;
                    if (dleft == 0) {
                        unsigned long long cl = 0;
                        if (lane == 0) cl = atomicAdd(gctr, 2ull);
                        dnext = dyn_from + (int64_t)__shfl_sync(0xFFFFFFFFu, cl, 0);
                        dleft = 2;
                    }
                    if (dnext >= ngroups) break;
                    g0 = dnext * 128;
                    ++dnext;
                    --dleft;
                }
                const int64_t e4 = g0 + 4 * lane;
                uint4 P, I, C[5] = {nP, nP, nP, nP, nP};
                if constexpr (kSelPrefetch) {
                    P = nP;
                    I = nI;
#pragma unroll
                    for (int v = 0; v < 5; ++v) C[v] = nC[v];
                    if (g0 + gstride < n_pad) load(g0 + gstride, nP, nI, nC);
                } else {
                    load(g0, P, I, C);
                }
                uint32_t c[20];
#pragma unroll
                for (int v = 0; v < 5; ++v) {
                    const bool z = POLICY == CACHE_POLICY_FIFO;
                    c[4 * v] = z ? 0u : C[v].x; c[4 * v + 1] = z ? 0u : C[v].y;
                    c[4 * v + 2] = z ? 0u : C[v].z; c[4 * v + 3] = z ? 0u : C[v].w;
                }
                const uint32_t pm[4] = {P.x, P.y, P.z, P.w}, pid[4] = {I.x, I.y, I.z, I.w};
                if constexpr (GRAN == CACHE_EVICT_ITEM) {
                    sweep_items_v4<POLICY>(a, kv, lim, mode, L, e4, pm, pid, c, sh, run, kmin, lane);
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        uint32_t col[CACHE_MAX_K];
#pragma unroll
                        for (int j = 0; j < CACHE_MAX_K; ++j) col[j] = j < 5 ? c[5 * q + j] : 0u;
                        sel_slot<POLICY, GRAN>(a, 5, kv, mode, L, e4 + q, pm[q], pid[q], col, sh, run, kmin, lane);
                    }
                }
                if (!in_dyn) {
                    g0 += gstride;
                    if (g0 >= dyn_from * 128) in_dyn = true;
                }
            }
        } else {
            for (int64_t e0 = ((int64_t)blockIdx.x * (kSelThreads / 32) + warp) * 32; e0 < n_pad;
                 e0 += (int64_t)gridDim.x * kSelThreads) {
                const int64_t e = e0 + lane;
                const uint32_t m = a.present[e];   // e < n_pad <= the padded capacity
                const uint32_t id = a.ids[e];
                uint32_t col[CACHE_MAX_K];
#pragma unroll
                for (int j = 0; j < CACHE_MAX_K; ++j)
                    col[j] = (POLICY != CACHE_POLICY_FIFO && j < nk) ? colp[e * nk + j] : 0u;
                sel_slot<POLICY, GRAN>(a, nk, kv, mode, L, e, m, id, col, sh, run, kmin, lane);
            }
        }
        run.flush(sh);
    };
    auto cand_sweep = [&](int mode, const SelLevel& L, int64_t nc) {
        const int64_t cper = (((nc + gridDim.x - 1) / gridDim.x) + 31) & ~(int64_t)31;
        const int64_t c0 = (int64_t)blockIdx.x * cper, c1 = min(nc, c0 + cper);
        DigitRun run;
        // item-mode apply: the evicted-key list only if the bitmap can miss a key (the host side
        // then sorts it); counts summed per CTA, one global atomic per CTA
        const bool ev_list = a.ev_cap && !(L.ev_lim && L.T >= L.kb && L.T - L.kb < L.ev_lim);
        uint32_t nev = 0, ndirty = 0;
        for (int64_t i0 = c0 + warp * 32; i0 < c1; i0 += kSelThreads) {
            const int64_t i = i0 + lane;
            if (GRAN == CACHE_EVICT_ITEM && mode == kSweepFinal)
                cand_apply_item(a, km.num_k, L, i, i < c1, lane, ev_list, nev, ndirty);
            else
                sel_cand<POLICY, GRAN>(a, km, mode, L, i, i < c1, sh, run, lane);
        }
        run.flush(sh);
        if (GRAN == CACHE_EVICT_ITEM && mode == kSweepFinal) {
            __shared__ unsigned long long s_cnt[2];
            if (threadIdx.x < 2) s_cnt[threadIdx.x] = 0ull;
            __syncthreads();
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) {
                nev += __shfl_xor_sync(0xFFFFFFFFu, nev, o);
                ndirty += __shfl_xor_sync(0xFFFFFFFFu, ndirty, o);
            }
            if (lane == 0) {
                if (nev) atomicAdd(&s_cnt[0], (unsigned long long)nev);
                if (ndirty) atomicAdd(&s_cnt[1], (unsigned long long)ndirty);
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                if (s_cnt[0]) atomicAdd(&a.out->cnt[0], s_cnt[0]);
                if (s_cnt[1]) atomicAdd(&a.out->cnt[1], s_cnt[1]);
            }
        }
    };

    // final apply (the candidates <= T, or one more full sweep), then the ordered lists
    auto finish = [&](SelLevel L, bool compacted, int64_t ncand, bool fail, int level, int full,
                      int compact_level, int* tsp = nullptr, uint32_t window = 0u) {
        int ts_dummy = 0;
        int& ts = tsp ? *tsp : ts_dummy;
        unsigned long long kmin_unused = ~0ull;
        L.T = L.lo + ((1ull << L.w) - 1ull);
        if (!fail) {
            if (compacted) {
                cand_sweep(kSweepFinal, L, ncand);
            } else {
                full_sweep(kSweepFinal, L, kmin_unused);
                ++full;
            }
        }
        sel_stamp(ts);
        grid.sync();   // every apply is done: the bitmaps and the evicted-key list are complete
        sel_stamp(ts);
        bool ev_sorted = false;
        if (!fail) {
            // evicted keys (unique): marked in the bitmap over [kb, kb + ev_lim) as they went;
            // sorted by the compaction below unless one fell beyond it (then the host side sorts)
            const unsigned long long kb = L.kb;
            ev_sorted = L.ev_lim && L.T >= kb && __ldcg(&a.out->ev_over) == 0u;
            const BitJob jobs[4] = {
                BitJob{a.dslot_bits, a.dslot_words, a.dirty_slot, 1ull, 0ull, nullptr, 0ull},
                BitJob{a.did_bits, a.did_words, a.dirty_id, (unsigned long long)a.world, (unsigned long long)a.rank,
                       nullptr, 0ull},
                BitJob{a.pool_bits, a.pool_words, a.ev_pool, 1ull, 0ull, nullptr, 0ull},
                // every evicted key lies in [kb, kb + ev_lim) (no overflow); T itself may lie beyond
                BitJob{ev_sorted ? a.ev_bits : nullptr,
                       ev_sorted ? (int64_t)min((L.T - kb) / 32 + 1, (unsigned long long)a.ev_bits_words) : 0,
                       a.ev_sorted, 1ull, kb, a.ev_masked, a.ev_mask}};
            compact_bitmaps<4>(jobs, a.part, grid, ts);
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            a.out->window = window;
            a.out->T = L.T;
            a.out->levels = (uint32_t)level;
            a.out->full_sweeps = (uint32_t)full;
            a.out->compact_level = (uint32_t)compact_level;
            a.out->err = fail ? 1u : 0u;
            a.out->ev_sorted = ev_sorted ? 1u : 0u;
        }
    };
    auto kmin_to_global = [&](unsigned long long kmin) {
        unsigned long long inv = ~kmin;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            const unsigned long long y = shfl_xor_u64(inv, o);
            inv = y > inv ? y : inv;
        }
        if (lane == 0 && inv) atomicMax(&a.out->kmin_inv, inv);
    };

    // Single-sweep window estimate: a block sample of this shard (every S-th 32-slot block, a
    // warp per block) -> the upper bin edge of the sample rank of the target-th key, padded;
    // sets L.T = that edge and L.compact (the level-0 sweep then compacts every key below it).
    auto window_estimate = [&](SelLevel& L, unsigned long long target, int& ts) {
        // every S-th block of 32 slots, a warp per block (lane = slot: every load a full line).
        // Single slots every S slots (random 4-B accesses) ran at a fraction of the HBM rate:
        // 15 us for the 1/63 sample of 12.5M slots (NV_SEL_TRACE)
        clear_sh();
        unsigned long long kdummy = ~0ull;
        DigitRun run;
        const uint32_t* colp = policy_col<POLICY>(a);
        const int64_t S = a.sample, nblk = (a.n_slots + 31) / 32, nw = (int64_t)gridDim.x * (kSelThreads / 32);
        for (int64_t bi = (int64_t)blockIdx.x * (kSelThreads / 32) + warp; bi * S < nblk; bi += nw) {
            const int64_t e = bi * S * 32 + lane;   // e < the 256-padded capacity
            const uint32_t m = e < a.n_slots ? __ldcg(a.present + e) : 0u, id = __ldcg(a.ids + e);
            uint32_t col[CACHE_MAX_K];
#pragma unroll
            for (int j = 0; j < CACHE_MAX_K; ++j)
                col[j] = (POLICY != CACHE_POLICY_FIFO && j < nk) ? __ldcg(colp + e * nk + j) : 0u;
            sel_slot<POLICY, GRAN>(a, nk, kv, kSweepL0, L, e, m, id, col, sh, run, kdummy, lane);
        }
        run.flush(sh);
        sel_stamp(ts);
        flush_sh(a.hist_s);
        grid.sync();
        sel_stamp(ts);
        const unsigned long long ns = sel_total(a.hist_s);
        if (ns && a.units) {
            // pad: 4 sigma of the sampling noise + two sample blocks' worth of units (on keys
            // that grow with the slot, a 32-slot block is the sample's resolution)
            const double r = ceil((double)target * (double)ns / (double)a.units);
            const unsigned long long rhi =
                (unsigned long long)(r + 4.0 * sqrt(r) + 64.0 * (GRAN == CACHE_EVICT_ITEM ? nk : 1) + 16.0);
            if (rhi <= ns) {
                const PickRes ps = sel_pick(a.hist_s, rhi);
                unsigned long long lo_s = 0;
                int w_s = 0;
                if (ps.bin < (uint32_t)kSelBins) {
                    sel_bin0_range(ps.bin, lo_s, w_s);
                    const unsigned long long hi = lo_s + (1ull << w_s);
                    if (hi > lo_s) { L.T = hi; L.compact = true; }   // not past 2^64
                }
            }
        }
        sel_stamp(ts);
    };
    // ---- distributed phases: one level per launch, the state in a.state ----
    if (a.phase == kPhaseL0) {
        SelLevel L{0ull, 0ull, 64, 0, false, 0ull, 0ull};
        // the window on this shard: its share of the n keys taken as n / world (ids, hence
        // keys, interleave over the ranks); whether the window holds is decided per rank by
        // the level-0 pick (k_evict_dpick) -- a rank whose window misses sweeps again
        int ts_unused = 0;
        if (a.sample > 0) window_estimate(L, (a.n + (unsigned long long)a.world - 1ull) / (unsigned long long)a.world, ts_unused);
        if (blockIdx.x == 0 && threadIdx.x == 0) a.out->whi = L.compact ? L.T : 0ull;
        clear_sh();
        unsigned long long kmin = ~0ull;
        full_sweep(kSweepL0, L, kmin);
        flush_sh(a.level_hist);
        kmin_to_global(kmin);
        return;
    }
    if (a.phase == kPhaseLevel || a.phase == kPhaseFinal) {
        const SelState S = *a.state;
        SelLevel L{S.lo, 0ull, S.w, S.shift, false, S.kb, S.ev_lim};
        if (a.phase == kPhaseFinal) {
            int ts_unused = 0;
            finish(L, S.compacted != 0u, S.ncand, S.fail != 0u, (int)S.level, (int)S.full, (int)S.compact_level,
                   &ts_unused, S.pad1);
            return;
        }
        if (S.done) return;
        L.compact = !S.compacted && S.pcnt <= a.cand_cap;
        clear_sh();
        unsigned long long kmin = ~0ull;
        if (!S.compacted) full_sweep(kSweepLevel, L, kmin);
        else cand_sweep(kSweepLevel, L, S.ncand);
        flush_sh(a.level_hist);
        return;
    }

    // ---- single cache: the whole selection in this launch ----
    // level 0: log-bin histogram + min key
    int ts = 0;
    sel_stamp(ts);
    SelLevel L{0ull, 0ull, 64, 0, false, 0ull, 0ull};
    // Single-sweep window: a systematic 1/S sample of the slots estimates the n-th key; its
    // rank r = n * (sampled units / live units) is padded by 4 sqrt(r) + 16, and the upper edge
    // of the sample bin holding that rank becomes the window hi.  The level-0 sweep then also
    // compacts every key < hi.  If the n-th key's level-0 bin ends below hi (and nothing
    // overflowed the buffer), every key the selection can still pick is a candidate: the levels
    // and the apply run on the candidates and the second full sweep is skipped.  Otherwise the
    // usual path runs -- the estimate only decides speed, never the result.
    if (a.sample > 0) window_estimate(L, a.n, ts);
    clear_sh();
    unsigned long long kmin = ~0ull;
    full_sweep(kSweepL0, L, kmin);
    sel_stamp(ts);
    flush_sh(a.hist);
    kmin_to_global(kmin);
    grid.sync();
    sel_stamp(ts);
    const bool windowed = L.compact;
    const unsigned long long whi = L.T;
    L.compact = false;
    L.T = 0ull;
    L.kb = ~__ldcg(&a.out->kmin_inv);
    L.ev_lim = a.ev_bits ? (unsigned long long)a.ev_bits_words * 32ull : 0ull;
    PickRes p = sel_pick(a.hist, a.n);
    bool fail = p.bin >= (uint32_t)kSelBins;
    unsigned long long rem = a.n - p.before;
    sel_bin0_range(p.bin, L.lo, L.w);
    bool done = fail || p.cnt == rem || L.w == 0;
    bool compacted = false;
    int64_t ncand = 0;
    int level = 1, full = 1, compact_level = 0;
    uint32_t window = 0;
    if (windowed) {
        const unsigned long long nw = __ldcg(&a.out->cnt_w);
        // T <= lo + 2^w - 1 whatever the levels pick: inside the window iff that is < whi
        if (!fail && nw <= a.cand_cap && L.lo + ((1ull << L.w) - 1ull) < whi) {
            compacted = true;
            ncand = (int64_t)nw;
            window = 1;
        } else {
            window = 2;
        }
    }
    while (!done) {
        const int D = L.w < 12 ? L.w : 12;
        L.shift = L.w - D;
        clear_sh();
        if (!compacted) {
            L.compact = p.cnt <= a.cand_cap;
            full_sweep(kSweepLevel, L, kmin);
            ++full;
        } else {
            L.compact = false;
            cand_sweep(kSweepLevel, L, ncand);
        }
        sel_stamp(ts);
        uint32_t* gh = a.hist + (size_t)(level < kSelMaxLevels ? level : kSelMaxLevels - 1) * kSelBins;
        flush_sh(gh);
        grid.sync();
        sel_stamp(ts);
        if (L.compact) {
            compacted = true;
            ncand = (int64_t)__ldcg(&a.out->cnt[3]);
            compact_level = level;
        }
        p = sel_pick(gh, rem);
        if (p.bin >= (uint32_t)kSelBins || level + 1 >= kSelMaxLevels) { fail = true; break; }
        L.lo += (unsigned long long)p.bin << L.shift;
        L.w = L.shift;
        rem -= p.before;
        done = p.cnt == rem || L.w == 0;
        ++level;
    }
    sel_stamp(ts);
    finish(L, compacted, ncand, fail, level, full, compact_level, &ts, window);
    sel_stamp(ts);
}

// Pick of one distributed level (one CTA): the single-cache kernel's pick arithmetic on the
// rank-summed histogram, applied to the state in device memory (every rank reaches the same
// state from the same histogram).
__global__ void __launch_bounds__(kSelThreads) k_evict_dpick(SelArgs a, const uint32_t* ghist, int level) {
    __shared__ SelState S;
    if (threadIdx.x == 0) S = *a.state;
    __syncthreads();
    if (level > 0 && (S.done || S.fail)) return;   // block-uniform
    if (level == 0) {
        const PickRes p = sel_pick(ghist, a.n);
        if (threadIdx.x == 0) {
            S.kb = ~__ldcg(&a.out->kmin_inv);   // this rank's own min key: the base of its lists
            S.ev_lim = a.ev_bits ? (unsigned long long)a.ev_bits_words * 32ull : 0ull;
            S.fail = p.bin >= (uint32_t)kSelBins;
            S.rem = a.n - p.before;
            S.pcnt = p.cnt;
            sel_bin0_range(p.bin, S.lo, S.w);
            S.done = S.fail || p.cnt == S.rem || S.w == 0;
            S.compacted = 0u;
            S.ncand = 0;
            S.level = 1u;
            S.full = 1u;
            S.compact_level = 0u;
            S.pad1 = 0u;   // single-sweep window: 0 off, 1 this rank's candidates hold the cut, 2 missed
            const unsigned long long whi = __ldcg(&a.out->whi), nw = __ldcg(&a.out->cnt_w);
            if (whi) {
                if (!S.fail && S.lo + ((1ull << S.w) - 1ull) < whi && nw <= a.cand_cap) {
                    S.compacted = 1u;
                    S.ncand = (long long)nw;
                    S.pad1 = 1u;
                } else {
                    S.pad1 = 2u;
                }
            }
        }
    } else {
        // this level's sweep compacted iff the state allowed it before the sweep (same rule)
        const bool compacted_now = !S.compacted && S.pcnt <= a.cand_cap;
        const PickRes p = sel_pick(ghist, S.rem);
        if (threadIdx.x == 0) {
            if (!S.compacted) S.full++;
            if (compacted_now) {
                S.compacted = 1u;
                S.ncand = (long long)__ldcg(&a.out->cnt[3]);
                S.compact_level = (uint32_t)level;
            }
            if (p.bin >= (uint32_t)kSelBins || S.level + 1 >= (uint32_t)kSelMaxLevels) {
                S.fail = 1u;
                S.done = 1u;
            } else {
                S.lo += (unsigned long long)p.bin << S.shift;
                S.w = S.shift;
                S.rem -= p.before;
                S.pcnt = p.cnt;
                S.done = p.cnt == S.rem || S.w == 0;
                S.level++;
            }
        }
    }
    if (threadIdx.x == 0) {
        if (!S.done) S.shift = S.w - (S.w < 12 ? S.w : 12);   // the next level's digit
        *a.state = S;
    }
}

template <int POLICY, int GRAN, bool NK5>
static cudaError_t launch_select_t(const SelArgs& a, const KMap& km, cudaStream_t s) {
    static int wave = [] {
        int bps = 0, dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const int dyn0 = NK5 ? (kSelStaged ? kStages * kStageBytes : (kSelCpAsync ? kCpRingBytes : (kSelColT ? kColTBytes : 0)))
                             : 0;
        if (dyn0 > 0)
            cudaFuncSetAttribute(k_evict_select<POLICY, GRAN, NK5>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn0);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_evict_select<POLICY, GRAN, NK5>, kSelThreads, dyn0) !=
                cudaSuccess ||
            bps < 1)
            bps = 1;
        return bps * sms;
    }();
    // |K| = 5: a lane takes 4 slots per group, so a CTA covers 4 x kSelThreads slots per pass --
    // small caches get no idle CTAs (each grid barrier costs more with more CTAs: C2's 100K
    // slots ran 196 CTAs, of which 3/4 had no slot)
    const int64_t per_cta = NK5 ? 4 * kSelThreads : kSelThreads;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(wave, (a.n_slots + per_cta - 1) / per_cta));
    SelArgs aa = a;
    KMap kk = km;
    void* args[] = {&aa, &kk};
    const size_t dyn = NK5 ? (kSelStaged ? (size_t)kStages * kStageBytes
                                         : (kSelCpAsync ? (size_t)kCpRingBytes : (kSelColT ? (size_t)kColTBytes : 0)))
                           : 0;
    return cudaLaunchCooperativeKernel((const void*)k_evict_select<POLICY, GRAN, NK5>, grid, kSelThreads, args, dyn, s);
}

void sel_trace_reset(cudaStream_t s) {
    static unsigned long long lo[kSelTraceN], hi[kSelTraceN];
    for (int i = 0; i < kSelTraceN; ++i) { lo[i] = ~0ull; hi[i] = 0ull; }
    cudaMemcpyToSymbolAsync(g_sel_tmin, lo, sizeof(lo), 0, cudaMemcpyHostToDevice, s);
    cudaMemcpyToSymbolAsync(g_sel_tmax, hi, sizeof(hi), 0, cudaMemcpyHostToDevice, s);
}
int sel_trace_read(unsigned long long* tmin, unsigned long long* tmax, unsigned long long* cta) {
    cudaMemcpyFromSymbol(tmin, g_sel_tmin, sizeof(unsigned long long) * kSelTraceN);
    cudaMemcpyFromSymbol(tmax, g_sel_tmax, sizeof(unsigned long long) * kSelTraceN);
    if (cta) cudaMemcpyFromSymbol(cta, g_sel_cta, sizeof(unsigned long long) * kSelTraceCta * 1024);
    return NV_SEL_TRACE != 0 ? kSelTraceN : 0;
}

cudaError_t launch_evict_dpick(const SelArgs& a, const uint32_t* ghist, int level, cudaStream_t s) {
    k_evict_dpick<<<1, kSelThreads, 0, s>>>(a, ghist, level);
    return cudaGetLastError();
}

cudaError_t launch_evict_select(const SelArgs& a, const KMap& km, cudaStream_t s) {
    cudaError_t r = cudaSuccess;
#define NV_SEL(P, G) r = km.num_k == 5 ? launch_select_t<P, G, true>(a, km, s) : launch_select_t<P, G, false>(a, km, s)
    NV_EVICT_DISPATCH(NV_SEL);
#undef NV_SEL
    return r;
}

}  // namespace nv
