// sort.cu -- ascending LSD radix sort of 64-bit keys on the GPU.  Used for cache_evict's
// out_evicted (the selected items in eviction = key order, R11 / R24): the selection kernels
// emit keys in arbitrary order and sorting ~10^5-10^6 keys on the host cost tens of ms.
//
// ceil(bits / 8) passes of 8-bit digits over (key - base), so a list whose keys span a narrow
// range (evicted keys: [min key, threshold]; slots: [0, hwm)) needs only the passes that range
// has; every pass is stable:
//   k_sort_count    per 2,048-key tile: digit counts (warp-aggregated shared atomics),
//                   stored digit-major counts[d][tile], and the pass's digit totals
//   k_sort_scan     one CTA per digit d: base = sum of the lower digits' totals, then a
//                   block-parallel exclusive scan over the tiles -> the output position of
//                   each tile's first key with digit d
//   k_sort_scatter  the tile again in 8 rounds of 256 keys (index order): rank within the warp
//                   from __match_any_sync, prefix over the warps per digit, running base per
//                   digit across rounds -> every key lands after all earlier keys of its digit
#include <cooperative_groups.h>

#include "kernels.h"

namespace nv {

constexpr int kSortThreads = 256, kSortRounds = 8, kSortTile = kSortThreads * kSortRounds;

__global__ void __launch_bounds__(256)
k_sort_count(const unsigned long long* __restrict__ keys, int64_t n, int shift, unsigned long long kbase,
             uint32_t* __restrict__ counts, int64_t ntiles, uint32_t* __restrict__ dtot) {
    __shared__ uint32_t sh[256];
    sh[threadIdx.x] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t base = (int64_t)blockIdx.x * kSortTile;
    for (int r = 0; r < kSortRounds; ++r) {
        const int64_t i = base + r * kSortThreads + threadIdx.x;
        const bool v = i < n;
        const unsigned d = v ? (unsigned)(((keys[i] - kbase) >> shift) & 255ull) : 256u;
        const unsigned peers = __match_any_sync(0xFFFFFFFFu, d);
        if (v && lane == __ffs(peers) - 1) atomicAdd(&sh[d], (unsigned)__popc(peers));
    }
    __syncthreads();
    const uint32_t c = sh[threadIdx.x];
    counts[(int64_t)threadIdx.x * ntiles + blockIdx.x] = c;
    if (c) atomicAdd(&dtot[threadIdx.x], c);
}

__device__ __forceinline__ uint32_t block_incl_scan_1024(uint32_t x, uint32_t* ws, uint32_t* total) {
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) ws[w] = x;
    __syncthreads();
    if (w == 0) {
        uint32_t v = ws[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, v, o);
            if (lane >= o) v += y;
        }
        ws[lane] = v;
    }
    __syncthreads();
    const uint32_t r = x + (w ? ws[w - 1] : 0u);
    *total = ws[31];
    __syncthreads();
    return r;
}

// CTA d: counts[d][0..ntiles) -> exclusive positions, offset by the keys of all digits < d.
__global__ void __launch_bounds__(1024) k_sort_scan(uint32_t* __restrict__ counts, int64_t ntiles,
                                                    const uint32_t* __restrict__ dtot) {
    __shared__ uint32_t ws[32];
    const int d = blockIdx.x, t = threadIdx.x;
    uint32_t tot = 0;
    uint32_t lower = (t < d) ? dtot[t] : 0u;   // 256 digits <= 1024 threads
    uint32_t run = block_incl_scan_1024(lower, ws, &tot);
    (void)run;
    uint32_t carry = tot;                      // sum over digits < d
    uint32_t* a = counts + (int64_t)d * ntiles;
    for (int64_t i0 = 0; i0 < ntiles; i0 += 1024) {
        const int64_t i = i0 + t;
        const uint32_t c = i < ntiles ? a[i] : 0u;
        uint32_t blk = 0;
        const uint32_t incl = block_incl_scan_1024(c, ws, &blk);
        if (i < ntiles) a[i] = carry + incl - c;
        carry += blk;
    }
}

__global__ void __launch_bounds__(256)
k_sort_scatter(const unsigned long long* __restrict__ in, unsigned long long* __restrict__ out, int64_t n, int shift,
               unsigned long long kbase, const uint32_t* __restrict__ offs, int64_t ntiles) {
    __shared__ uint32_t s_base[256];
    __shared__ uint32_t s_tot[256];
    __shared__ uint32_t s_w[8][256];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    s_base[threadIdx.x] = offs[(int64_t)threadIdx.x * ntiles + blockIdx.x];
    const int64_t base = (int64_t)blockIdx.x * kSortTile;
    for (int r = 0; r < kSortRounds; ++r) {
#pragma unroll
        for (int w = 0; w < 8; ++w) s_w[w][threadIdx.x] = 0u;
        __syncthreads();
        const int64_t i = base + r * kSortThreads + threadIdx.x;
        const bool v = i < n;
        const unsigned long long k = v ? in[i] : 0ull;
        const unsigned d = v ? (unsigned)(((k - kbase) >> shift) & 255ull) : 256u;
        const unsigned peers = __match_any_sync(0xFFFFFFFFu, d);
        const unsigned rank = (unsigned)__popc(peers & ((1u << lane) - 1u));
        if (v && lane == __ffs(peers) - 1) s_w[warp][d] = (unsigned)__popc(peers);
        __syncthreads();
        {   // thread = digit: exclusive prefix over the warps (warp order = index order)
            uint32_t run = 0;
#pragma unroll
            for (int w = 0; w < 8; ++w) {
                const uint32_t c = s_w[w][threadIdx.x];
                s_w[w][threadIdx.x] = run;
                run += c;
            }
            s_tot[threadIdx.x] = run;
        }
        __syncthreads();
        if (v) out[(int64_t)s_base[d] + s_w[warp][d] + rank] = k;
        __syncthreads();
        s_base[threadIdx.x] += s_tot[threadIdx.x];
    }
}

// scratch: counts[256][ntiles] | digit totals [8 passes][256]
int64_t sort_scratch_words(int64_t n) { return 256 * std::max<int64_t>(1, (n + kSortTile - 1) / kSortTile) + 8 * 256; }

// Small lists: one CTA per list sorts up to kSmallSort keys in shared memory (bitonic network
// over the next power of two, padding = all-ones keys) -- one launch for several lists instead
// of 3 launches per radix pass each.
__global__ void __launch_bounds__(1024) k_sort_small(SortSegs segs) {
    extern __shared__ unsigned long long sk[];
    const SortSeg sg = segs.s[blockIdx.x];
    const int n = (int)sg.n;
    int N = 2;
    while (N < n) N <<= 1;
    for (int i = threadIdx.x; i < N; i += blockDim.x) sk[i] = i < n ? sg.keys[i] : ~0ull;
    __syncthreads();
    for (int k = 2; k <= N; k <<= 1) {
        for (int j = k >> 1, lj = __ffs(j) - 1; j > 0; j >>= 1, --lj) {
            for (int p = threadIdx.x; p < N / 2; p += blockDim.x) {
                const int i = ((p >> lj) << (lj + 1)) | (p & (j - 1)), ixj = i + j;   // j is a power of 2
                const unsigned long long a = sk[i], b = sk[ixj];
                if ((a > b) == ((i & k) == 0)) { sk[i] = b; sk[ixj] = a; }
            }
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) sg.keys[i] = sk[i];
}

void launch_sort_small(const SortSegs& segs, cudaStream_t s) {
    if (segs.k <= 0) return;
    static bool attr = (cudaFuncSetAttribute(k_sort_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             kSmallSort * 8), true);
    (void)attr;
    int64_t mx = 2;
    for (int i = 0; i < segs.k; ++i) mx = std::max<int64_t>(mx, segs.s[i].n);
    int N = 2;
    while (N < mx) N <<= 1;
    k_sort_small<<<segs.k, 1024, (size_t)N * 8, s>>>(segs);
}

unsigned long long* launch_sort_u64(unsigned long long* keys, unsigned long long* tmp, int64_t n, uint32_t* scratch,
                                    cudaStream_t s, int bits, unsigned long long base) {
    if (n <= 1) return keys;
    const int passes = (std::min(64, std::max(1, bits)) + 7) / 8;
    const int64_t ntiles = (n + kSortTile - 1) / kSortTile;
    unsigned long long *src = keys, *dst = tmp;
    uint32_t* dtot = scratch + 256 * ntiles;
    cudaMemsetAsync(dtot, 0, 8 * 256 * sizeof(uint32_t), s);
    for (int pass = 0; pass < passes; ++pass) {
        const int shift = 8 * pass;
        k_sort_count<<<(unsigned)ntiles, 256, 0, s>>>(src, n, shift, base, scratch, ntiles, dtot + 256 * pass);
        k_sort_scan<<<256, 1024, 0, s>>>(scratch, ntiles, dtot + 256 * pass);
        k_sort_scatter<<<(unsigned)ntiles, 256, 0, s>>>(src, dst, n, shift, base, scratch, ntiles);
        std::swap(src, dst);
    }
    return src;   // the buffer holding the sorted keys (keys for an even number of passes)
}

// ---- one cooperative launch for several long lists: the same three steps per pass as the
// kernels above (tile counts, per-digit scan over the tiles, stable scatter), separated by grid
// barriers instead of kernel boundaries (3 launches per pass per list -> 1 launch in all; the
// eviction's lists of ~10^5-10^6 keys were launch- and tail-bound at ~25 us per pass). ----
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t block_scan_incl(uint32_t x, uint32_t* ws, uint32_t* total) {
    const int t = threadIdx.x, lane = t & 31, w = t >> 5, nw = (int)(blockDim.x >> 5);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) ws[w] = x;
    __syncthreads();
    if (w == 0) {
        uint32_t v = lane < nw ? ws[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, v, o);
            if (lane >= o) v += y;
        }
        ws[lane] = v;
    }
    __syncthreads();
    const uint32_t r = x + (w ? ws[w - 1] : 0u);
    *total = ws[nw - 1];
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(256) k_sort_coop(SortJobs J, uint32_t* __restrict__ scratch, int64_t max_tiles) {
    __shared__ uint32_t sh[256];
    __shared__ uint32_t s_base[256];
    __shared__ uint32_t s_tot[256];
    __shared__ uint32_t s_w[8][256];
    __shared__ uint32_t ws[32];
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t* counts = scratch;                                // [256][max_tiles]
    uint32_t* dtot_all = scratch + 256 * max_tiles;            // [4 jobs][8 passes][256]
    for (int i = blockIdx.x * 256 + threadIdx.x; i < 4 * 8 * 256; i += gridDim.x * 256) dtot_all[i] = 0u;
    grid.sync();
    for (int jb = 0; jb < J.k; ++jb) {
        const SortJob job = J.j[jb];
        const int64_t n = job.n, ntiles = (n + kSortTile - 1) / kSortTile;
        unsigned long long *src = job.keys, *dst = job.tmp;
        for (int pass = 0; pass < job.passes; ++pass) {
            const int shift = 8 * pass;
            uint32_t* dtot = dtot_all + (jb * 8 + pass) * 256;
            // 1. per-tile digit counts
            for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                sh[threadIdx.x] = 0;
                __syncthreads();
                const int64_t base = tile * kSortTile;
                for (int r = 0; r < kSortRounds; ++r) {
                    const int64_t i = base + r * kSortThreads + threadIdx.x;
                    const bool v = i < n;
                    const unsigned d = v ? (unsigned)(((src[i] - job.base) >> shift) & 255ull) : 256u;
                    const unsigned peers = __match_any_sync(0xFFFFFFFFu, d);
                    if (v && lane == __ffs(peers) - 1) atomicAdd(&sh[d], (unsigned)__popc(peers));
                }
                __syncthreads();
                const uint32_t c = sh[threadIdx.x];
                counts[(int64_t)threadIdx.x * ntiles + tile] = c;
                if (c) atomicAdd(&dtot[threadIdx.x], c);
                __syncthreads();
            }
            grid.sync();
            // 2. digit d: exclusive positions over the tiles, offset by the lower digits' keys
            for (int d = blockIdx.x; d < 256; d += gridDim.x) {
                uint32_t tot = 0;
                (void)block_scan_incl(threadIdx.x < d ? __ldcg(dtot + threadIdx.x) : 0u, ws, &tot);
                uint32_t carry = tot;
                uint32_t* a = counts + (int64_t)d * ntiles;
                for (int64_t i0 = 0; i0 < ntiles; i0 += 256) {
                    const int64_t i = i0 + threadIdx.x;
                    const uint32_t c = i < ntiles ? __ldcg(a + i) : 0u;
                    uint32_t blk = 0;
                    const uint32_t incl = block_scan_incl(c, ws, &blk);
                    if (i < ntiles) a[i] = carry + incl - c;
                    carry += blk;
                }
            }
            grid.sync();
            // 3. stable scatter
            for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                s_base[threadIdx.x] = __ldcg(counts + (int64_t)threadIdx.x * ntiles + tile);
                const int64_t base = tile * kSortTile;
                for (int r = 0; r < kSortRounds; ++r) {
#pragma unroll
                    for (int w = 0; w < 8; ++w) s_w[w][threadIdx.x] = 0u;
                    __syncthreads();
                    const int64_t i = base + r * kSortThreads + threadIdx.x;
                    const bool v = i < n;
                    const unsigned long long k = v ? src[i] : 0ull;
                    const unsigned d = v ? (unsigned)(((k - job.base) >> shift) & 255ull) : 256u;
                    const unsigned peers = __match_any_sync(0xFFFFFFFFu, d);
                    const unsigned rank = (unsigned)__popc(peers & ((1u << lane) - 1u));
                    if (v && lane == __ffs(peers) - 1) s_w[warp][d] = (unsigned)__popc(peers);
                    __syncthreads();
                    {
                        uint32_t run = 0;
#pragma unroll
                        for (int w = 0; w < 8; ++w) {
                            const uint32_t c = s_w[w][threadIdx.x];
                            s_w[w][threadIdx.x] = run;
                            run += c;
                        }
                        s_tot[threadIdx.x] = run;
                    }
                    __syncthreads();
                    if (v) dst[(int64_t)s_base[d] + s_w[warp][d] + rank] = k;
                    __syncthreads();
                    s_base[threadIdx.x] += s_tot[threadIdx.x];
                }
                __syncthreads();
            }
            grid.sync();
            unsigned long long* t = src;
            src = dst;
            dst = t;
        }
        if (src != job.keys) {   // odd number of passes: the lists share tmp, land in keys
            for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256)
                job.keys[i] = src[i];
            grid.sync();
        }
    }
}

int64_t sort_coop_scratch_words(int64_t max_n) {
    return 256 * std::max<int64_t>(1, (max_n + kSortTile - 1) / kSortTile) + 4 * 8 * 256;
}

cudaError_t launch_sort_coop(const SortJobs& jobs, uint32_t* scratch, cudaStream_t s) {
    if (jobs.k <= 0) return cudaSuccess;
    static int wave = [] {
        int bps = 0, dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_sort_coop, 256, 0) != cudaSuccess || bps < 1) bps = 1;
        return bps * sms;
    }();
    int64_t mt = 1;
    for (int i = 0; i < jobs.k; ++i) mt = std::max<int64_t>(mt, (jobs.j[i].n + kSortTile - 1) / kSortTile);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(wave, std::max<int64_t>(256, mt)));
    SortJobs jj = jobs;
    int64_t mtt = mt;
    void* args[] = {&jj, &scratch, &mtt};
    return cudaLaunchCooperativeKernel((const void*)k_sort_coop, grid, 256, args, 0, s);
}

__global__ void k_mask_u64(const unsigned long long* __restrict__ in, unsigned long long* __restrict__ out, int64_t n,
                           unsigned long long mask) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = in[i] & mask;
}

void launch_mask_u64(const unsigned long long* in, unsigned long long* out, int64_t n, unsigned long long mask,
                     cudaStream_t s) {
    if (n <= 0) return;
    const int grid = (int)std::min<int64_t>(1184, (n + 255) / 256);
    k_mask_u64<<<grid, 256, 0, s>>>(in, out, n, mask);
}

int sort_launches(int64_t n, int bits) { return n <= 1 ? 0 : 1 + 3 * ((std::min(64, std::max(1, bits)) + 7) / 8); }

}  // namespace nv
