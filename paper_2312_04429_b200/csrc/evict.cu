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

constexpr int kSelThreads = 512;

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
    constexpr int PER = kSelBins / kSelThreads;   // 8 bins per thread
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    uint32_t v[PER];
    const uint4* h4 = reinterpret_cast<const uint4*>(h + t * PER);
    const uint4 a = __ldcg(h4), b = __ldcg(h4 + 1);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
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

// Sweep modes (uniform over the grid within a phase)
enum { kSweepL0 = 0, kSweepLevel = 1, kSweepFinal = 2 };

struct SelLevel {
    unsigned long long lo, T;
    int w, shift;          // range [lo, lo + 2^w); digit = (key - lo) >> shift
    bool compact;
};

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

// One warp-aligned group of 32 entry slots (lane = one slot), every mode of a full sweep.
template <int POLICY, int GRAN>
__device__ __forceinline__ void sel_sweep_slot(const SelArgs& a, const KMap& km, const int (&kv)[CACHE_MAX_K],
                                               int mode, const SelLevel& L, int64_t e, bool valid, unsigned* sh,
                                               DigitRun& run, unsigned long long& kmin, int lane) {
    const int nk = km.num_k;
    const uint32_t m = valid ? a.present[e] : 0u;
    const uint32_t id = m ? a.ids[e] : 0u;
    if constexpr (GRAN == CACHE_EVICT_ENTRY) {
        const unsigned long long key = m ? entry_key<POLICY>(a.fcnt, a.lastacc, e, m, id, nk, kv) : 0ull;
        bool ev;
        sel_unit_common<POLICY, GRAN>(a, mode, L, key, m != 0u, (uint32_t)e, sh, run, kmin, lane, ev);
        if (mode == kSweepL0) return;
        const unsigned long long at = warp_claim(&a.out->cnt[0], ev, lane);
#pragma unroll
        for (int j = 0; j < CACHE_MAX_K; ++j) {
            if (j >= nk) break;   // warp-uniform
            const bool freed = ev && ((m >> j) & 1u);
            const unsigned long long pat = warp_claim(&a.out->cnt[2], freed, lane);
            if (freed && pat < a.pool_cap) a.ev_pool[pat] = (unsigned long long)(uint32_t)a.lslot[e * nk + j];
        }
        (void)warp_claim(&a.out->cnt[1], ev, lane);   // dirty count = evicted count in entry mode
        if (ev) {
            for (int j = 0; j < nk; ++j) a.fcnt[e * nk + j] = 0u;
            a.present[e] = 0u;
            a.inv_e[e] = __int_as_float(0x7FC00000);
            if (at < a.ev_cap && at < a.dirty_cap) {
                a.ev_key[at] = key;
                a.dirty_slot[at] = (unsigned long long)e;
                a.dirty_id[at] = id;
            }
        }
    } else {
        uint32_t keep = m;
#pragma unroll
        for (int j = 0; j < CACHE_MAX_K; ++j) {
            if (j >= nk) break;   // warp-uniform
            const bool has = (m >> j) & 1u;
            const unsigned long long key =
                has ? item_key(item_score<POLICY>(a.fcnt, a.lastacc, e * nk + j, kv[j]), id, j) : 0ull;
            bool ev;
            sel_unit_common<POLICY, GRAN>(a, mode, L, key, has, (uint32_t)e, sh, run, kmin, lane, ev);
            if (mode == kSweepL0) continue;
            const unsigned long long at = warp_claim(&a.out->cnt[0], ev, lane);
            if (ev) {
                keep &= ~(1u << j);
                if (at < a.ev_cap) {
                    a.ev_key[at] = key;
                    a.ev_pool[at] = (unsigned long long)(uint32_t)a.lslot[e * nk + j];
                }
                a.fcnt[e * nk + j] = 0u;
            }
        }
        if (mode == kSweepL0) return;
        const bool dirty = m && keep == 0u;
        if (keep != m) {
            a.present[e] = keep;
            if (dirty) a.inv_e[e] = __int_as_float(0x7FC00000);
        }
        const unsigned long long at = warp_claim(&a.out->cnt[1], dirty, lane);
        if (dirty && at < a.dirty_cap) {
            a.dirty_slot[at] = (unsigned long long)e;
            a.dirty_id[at] = id;
        }
    }
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
        const uint32_t m = ev ? a.present[e] : 0u;
#pragma unroll
        for (int j = 0; j < CACHE_MAX_K; ++j) {
            if (j >= nk) break;
            const bool freed = ev && ((m >> j) & 1u);
            const unsigned long long pat = warp_claim(&a.out->cnt[2], freed, lane);
            if (freed && pat < a.pool_cap) a.ev_pool[pat] = (unsigned long long)(uint32_t)a.lslot[e * nk + j];
        }
        (void)warp_claim(&a.out->cnt[1], ev, lane);
        if (ev) {
            for (int j = 0; j < nk; ++j) a.fcnt[e * nk + j] = 0u;
            a.present[e] = 0u;
            a.inv_e[e] = __int_as_float(0x7FC00000);
            if (at < a.ev_cap && at < a.dirty_cap) {
                a.ev_key[at] = key;
                a.dirty_slot[at] = (unsigned long long)e;
                a.dirty_id[at] = key & 0xFFFFFFFFull;
            }
        }
    } else {
        bool dirty = false;
        if (ev) {
            const int j = (int)(key & 7ull);
            const uint32_t bit = 1u << j;
            if (at < a.ev_cap) {
                a.ev_key[at] = key;
                a.ev_pool[at] = (unsigned long long)(uint32_t)a.lslot[e * nk + j];
            }
            a.fcnt[e * nk + j] = 0u;
            const uint32_t old = atomicAnd(a.present + e, ~bit);   // the entry's last bit -> dirty
            dirty = (old & ~bit) == 0u;
            if (dirty) a.inv_e[e] = __int_as_float(0x7FC00000);
        }
        const unsigned long long dat = warp_claim(&a.out->cnt[1], dirty, lane);
        if (dirty && dat < a.dirty_cap) {
            a.dirty_slot[dat] = (unsigned long long)e;
            a.dirty_id[dat] = (key >> 3) & 0xFFFFFFFFull;
        }
    }
}

template <int POLICY, int GRAN>
__global__ void __launch_bounds__(kSelThreads) k_evict_select(SelArgs a, KMap km) {
    __shared__ unsigned sh[kSelBins];
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int kv[CACHE_MAX_K];
#pragma unroll
    for (int j = 0; j < CACHE_MAX_K; ++j) kv[j] = km.kv[j];
    // this CTA's contiguous slice of the slots (warp-aligned)
    const int64_t per = (((a.n_slots + gridDim.x - 1) / gridDim.x) + 31) & ~(int64_t)31;
    const int64_t s0 = (int64_t)blockIdx.x * per, s1 = min(a.n_slots, s0 + per);

    auto clear_sh = [&]() {
        for (int i = threadIdx.x; i < kSelBins; i += kSelThreads) sh[i] = 0u;
        __syncthreads();
    };
    auto flush_sh = [&](uint32_t* gh) {
        __syncthreads();
        for (int i = threadIdx.x; i < kSelBins; i += kSelThreads)
            if (sh[i]) atomicAdd(gh + i, sh[i]);
    };
    auto full_sweep = [&](int mode, const SelLevel& L, unsigned long long& kmin) {
        DigitRun run;
        for (int64_t e0 = s0 + warp * 32; e0 < s1; e0 += kSelThreads) {
            const int64_t e = e0 + lane;
            sel_sweep_slot<POLICY, GRAN>(a, km, kv, mode, L, e, e < s1, sh, run, kmin, lane);
        }
        run.flush(sh);
    };
    auto cand_sweep = [&](int mode, const SelLevel& L, int64_t nc) {
        const int64_t cper = (((nc + gridDim.x - 1) / gridDim.x) + 31) & ~(int64_t)31;
        const int64_t c0 = (int64_t)blockIdx.x * cper, c1 = min(nc, c0 + cper);
        DigitRun run;
        for (int64_t i0 = c0 + warp * 32; i0 < c1; i0 += kSelThreads) {
            const int64_t i = i0 + lane;
            sel_cand<POLICY, GRAN>(a, km, mode, L, i, i < c1, sh, run, lane);
        }
        run.flush(sh);
    };

    // ---- level 0: log-bin histogram + min key ----
    SelLevel L{0ull, 0ull, 64, 0, false};
    clear_sh();
    unsigned long long kmin = ~0ull;
    full_sweep(kSweepL0, L, kmin);
    flush_sh(a.hist);
    {
        unsigned long long inv = ~kmin;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            const unsigned long long y = shfl_xor_u64(inv, o);
            inv = y > inv ? y : inv;
        }
        if (lane == 0 && inv) atomicMax(&a.out->kmin_inv, inv);
    }
    grid.sync();
    PickRes p = sel_pick(a.hist, a.n);
    bool fail = p.bin >= (uint32_t)kSelBins;
    unsigned long long rem = a.n - p.before;
    sel_bin0_range(p.bin, L.lo, L.w);
    bool done = fail || p.cnt == rem || L.w == 0;
    bool compacted = false;
    int64_t ncand = 0;
    int level = 1, full = 1, compact_level = 0;
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
        uint32_t* gh = a.hist + (size_t)(level < kSelMaxLevels ? level : kSelMaxLevels - 1) * kSelBins;
        flush_sh(gh);
        grid.sync();
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
    L.T = L.lo + ((1ull << L.w) - 1ull);
    if (!fail) {
        if (compacted) {
            cand_sweep(kSweepFinal, L, ncand);
        } else {
            full_sweep(kSweepFinal, L, kmin);
            ++full;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.out->T = L.T;
        a.out->levels = (uint32_t)level;
        a.out->full_sweeps = (uint32_t)full;
        a.out->compact_level = (uint32_t)compact_level;
        a.out->err = fail ? 1u : 0u;
    }
}

template <int POLICY, int GRAN>
static cudaError_t launch_select_t(const SelArgs& a, const KMap& km, cudaStream_t s) {
    static int wave = [] {
        int bps = 0, dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_evict_select<POLICY, GRAN>, kSelThreads, 0) !=
                cudaSuccess || bps < 1)
            bps = 1;
        return bps * sms;
    }();
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(wave, (a.n_slots + kSelThreads - 1) / kSelThreads));
    SelArgs aa = a;
    KMap kk = km;
    void* args[] = {&aa, &kk};
    return cudaLaunchCooperativeKernel((const void*)k_evict_select<POLICY, GRAN>, grid, kSelThreads, args, 0, s);
}

cudaError_t launch_evict_select(const SelArgs& a, const KMap& km, cudaStream_t s) {
    cudaError_t r = cudaSuccess;
#define NV_SEL(P, G) r = launch_select_t<P, G>(a, km, s)
    NV_EVICT_DISPATCH(NV_SEL);
#undef NV_SEL
    return r;
}

}  // namespace nv
