// cache.cu -- host engine behind the C ABI (include/nirvana_cache.h): storage layout in HBM,
// slot allocation, batch dispatch and error plumbing.  Every step of the lookup runs in the
// kernels of kernels.cu / score_tc.cu; this file only allocates, plans and launches.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <nvtx3/nvToolsExt.h>
#include <string>
#include <unordered_map>
#include <vector>
#include <iterator>

#include <unistd.h>

#include "kernels.h"

using namespace nv;

namespace {
thread_local std::string g_err = "no error";

// Exchange arena of the push path (identical geometry on every rank, so peers derive the
// offsets from the descriptor): flags | CTA counters | inv-norms | statuses | record inbox |
// bf16 query rows (rows padded to a multiple of 128 for the scan's TMA boxes).
struct ArenaLayout {
    size_t qflag, rflag, done, eflag, invq, qstat, inbox, qg, ehist, esel, total;
    int64_t rows;   // padded global rows
};
ArenaLayout arena_layout(int world, int64_t max_nb, int topk, int dim) {
    auto al = [](size_t x) { return (x + 1023) & ~size_t(1023); };
    ArenaLayout L{};
    L.rows = std::max<int64_t>(128, ((int64_t)world * max_nb + 127) / 128 * 128);
    L.qflag = 0;                          // u32[kMaxWorld]: query flag per sender
    L.rflag = 64;                         // u32[kMaxWorld]: record flag per sender
    L.done = 128;                         // u32[4]: CTA counters of the push kernels
    L.eflag = 256;                        // u32[8 passes][kMaxWorld]: eviction histogram flags
    size_t off = 1024;
    L.invq = off;  off = al(off + (size_t)L.rows * 4);
    L.qstat = off; off = al(off + (size_t)L.rows * 4);
    L.inbox = off; off = al(off + (size_t)world * max_nb * topk * sizeof(cache_shard_rec));
    L.qg = off;    off = al(off + (size_t)L.rows * dim * 2);
    L.ehist = off; off = al(off + 8 * 256 * 4);   // global eviction histogram per radix pass
    L.esel = off;  off = al(off + (size_t)kSelMaxLevels * kSelBins * 4);   // fused eviction: per level
    L.total = off;
    return L;
}

// cache_query_batch_host: batches of >= kHostSplitMin queries are uploaded in kHostSplit
// slices so the copy overlaps the scan (see cache_query_batch_host)
constexpr int kHostSplit = 4;
constexpr int64_t kHostSplitMin = 2048;
// cache_query_batch: tensor-core batches of >= kDevSplitMin queries are scanned in query
// slices so each slice's finalize + gather overlaps the next slice's scan (query_sliced)
// Measured (C2, 100K entries, b = 4,096): one launch 0.431 ms; 2 slices 0.444 ms (the
// concurrent finalize slows the scan 0.367 -> 0.388 ms, gaining back only the 22 us of the
// hidden gather), 3-4 slices 0.462 ms.  So auto = one launch; the option stays for callers
// whose gather is large relative to the scan (bigger latents, smaller caches).
constexpr int kDevSplitMax = 8;
constexpr int kDevSplitAuto = 1;
constexpr int64_t kEvBitsWords = 1 << 18;   // 1 MB: evicted keys spanning < 2^23 values are sorted in-kernel
constexpr int64_t kDevSplitMin = 2048;

cache_status fail(cache_status st, const std::string& msg) {
    g_err = msg;
    return st;
}

#define CK(call)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return fail(e_ == cudaErrorMemoryAllocation ? CACHE_E_OOM : CACHE_E_CUDA,         \
                        std::string(#call) + ": " + cudaGetErrorString(e_));                  \
    } while (0)

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    cudaError_t ensure(size_t need) {
        if (need <= n) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
        cudaError_t e = cudaMalloc(&p, std::max<size_t>(need, 1) * sizeof(T));
        if (e == cudaSuccess) n = need;
        return e;
    }
    // workspaces whose size creeps up call after call (eviction lists): grow by >= 1.25x so
    // the next call does not free + reallocate (cudaFree synchronises the device)
    cudaError_t ensure_grow(size_t need) { return need <= n ? cudaSuccess : ensure(std::max(need + need / 4, n + n / 4)); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
};

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// 2-D bf16 row-major [rows][dim] tensor map, box = 64 elements (128 B, swizzle-128B) x box_rows.
bool encode_rows(CUtensorMap* tm, const void* base, int64_t rows, int dim, int box_rows) {
    auto enc = get_encode();
    if (!enc) return false;
    cuuint64_t gdim[2] = {(cuuint64_t)dim, (cuuint64_t)rows};
    cuuint64_t gstride[1] = {(cuuint64_t)dim * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
    cuuint32_t estride[2] = {1, 1};
    CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), gdim, gstride, box,
                     estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}
}  // namespace

// NVTX range per public call (nsys / ncu --nvtx filter the library's phases; ~ns without a tool)
struct NvtxScope {
    explicit NvtxScope(const char* name) { nvtxRangePushA(name); }
    ~NvtxScope() { nvtxRangePop(); }
};

struct cache_t {
    cache_config cfg;
    int device = 0;
    int dim = 0, num_k = 0, sm_count = 148;
    int64_t cap = 0, cap_pad = 0, lcap = 0, L = 0;
    KMap km{};
    // HBM storage (SoA).  emb rows are 2*dim bytes (1,536 B at d=768), 128-B aligned.
    __nv_bfloat16* emb = nullptr;   // [cap_pad][dim]  stored x~ = bf16(x/||x||)
    float* inv_e = nullptr;         // [cap_pad]       f32(1/||x~||); NaN = empty / dirty slot
    uint32_t* ids = nullptr;        // [cap_pad]       entry id (insertion sequence)
    uint32_t* present = nullptr;    // [cap_pad]       bit j = K_j stored
    int32_t* lslot = nullptr;       // [cap_pad][num_k] latent-pool slot (-1 = hole)
    uint32_t* fcnt = nullptr;       // [cap_pad][num_k] LCBFU access counts f
    uint32_t* lastacc = nullptr;    // [cap_pad][num_k] batch clock of the last access (LRU)
    uint8_t* pool = nullptr;        // [lcap][L]       intermediate states
    CUtensorMap tm_e;               // TMA map of emb (box 64 x 256): single-CTA scan
    CUtensorMap tm_e128;            // TMA map of emb (box 64 x 128): CTA-pair scan (half a tile per CTA)
    bool tm_e_ok = false;
    // host mirrors / allocators
    // host mirror of the entry slots: live flag + id (allocation, high-water mark, inspection);
    // presence masks, latent slots and counters live on the device only
    std::vector<uint8_t> h_live;
    std::vector<uint32_t> h_ids;
    std::vector<int64_t> free_e, free_l;   // sorted descending: back() = lowest free slot
    int64_t hwm = 0, live_entries = 0, live_items = 0, queries = 0;
    uint64_t next_id = 0;
    uint32_t clock = 0;             // query batches so far (the LRU logical clock)
    int scorer = CACHE_SCORER_AUTO;
    int64_t launches = 0;
    cudaEvent_t prof[4] = {nullptr, nullptr, nullptr, nullptr};
    bool prof_on = false;
    // workspaces
    DevBuf<__nv_bfloat16> qbuf, ystage;
    DevBuf<float> invq, invstage;
    DevBuf<int32_t> qstat, istat;
    DevBuf<uint32_t> gk;   // per-query global k-th-best gate of the tcgen05 scorer
    DevBuf<Rec> recs;
    DevBuf<InsertPlan> iplan;
    DevBuf<CopyPlan> cplan;
    DevBuf<uint8_t> hq_in, hq_lat, hq_out;
    // pipelined host calls (cache_query_submit / _complete): per slot an input and an output
    // buffer on the device, pinned output staging, and the events of its last use
    struct AsyncSlot {
        DevBuf<uint8_t> in, out;
        void* h_out = nullptr;
        size_t h_out_n = 0;
        cudaEvent_t copied = nullptr, consumed = nullptr, done = nullptr;
        int64_t b = 0;
        int32_t topk = 0;
        bool pending = false;
    } aslot[2];
    // pinned host staging of an eviction's lists (keys, sorted keys, pool slots, entry slots,
    // dirty slots): reused across calls, so no pageable copies or fresh-page faults
    struct PinnedBuf {
        void* p = nullptr;
        size_t n = 0;
        cudaError_t ensure(size_t bytes) {
            if (bytes <= n) return cudaSuccess;
            // >= 1.25x growth: pinning is slow (tens of ms for tens of MB), and eviction sizes
            // creep up round after round
            bytes = std::max(bytes + bytes / 4, n + n / 4);
            if (p) cudaFreeHost(p);
            p = nullptr;
            n = 0;
            cudaError_t e = cudaHostAlloc(&p, std::max<size_t>(bytes, 64), cudaHostAllocDefault);
            if (e == cudaSuccess) n = bytes;
            return e;
        }
        void release() {
            if (p) cudaFreeHost(p);
            p = nullptr;
            n = 0;
        }
    } hev_sorted, hev_pool, hev_ds, hev_did;
    std::vector<int64_t> free_tmp;   // merge buffer of the free lists
    cudaEvent_t ev_first = nullptr;  // an eviction's pool / dirty-slot lists landed (host bookkeeping may start)
    void* h_out = nullptr;   // pinned staging of the packed host-call results
    size_t h_out_n = 0;
    // host-call pipeline: query H2D copies on their own stream, one event per sub-batch
    cudaStream_t hcopy = nullptr;
    cudaEvent_t hev[kHostSplit + 1] = {};
    // device query slices (query_sliced): finalize stream, one event per scanned slice + join
    int qslices = 0;   // 0 = auto (kDevSplitAuto for b >= kDevSplitMin), 1 = never, n = n slices
    cudaStream_t qside = nullptr;
    cudaEvent_t qev[kDevSplitMax + 1] = {};
    DevBuf<EvictState> est;
    DevBuf<unsigned int> ehist;
    DevBuf<unsigned long long> ekey, ekey2, ecnt;
    DevBuf<int64_t> eslot;         // entry slot of each evicted item
    DevBuf<uint32_t> escr;         // radix-sort scratch
    DevBuf<unsigned long long> epool;    // pool slot of each evicted item (sorted for the free list)
    DevBuf<unsigned long long> edirty, edid;   // dirty entries: slots, ids (each sorted on the GPU)
    DevBuf<unsigned long long> ckey;     // fused eviction (evict.cu): candidate keys / slots
    DevBuf<uint32_t> cslot;
    DevBuf<uint8_t> selws;               // per-level histograms + SelOut + compaction totals
    DevBuf<uint32_t> ebits;              // dirty-slot / dirty-id / freed-pool-slot / evicted-key bitmaps
    DevBuf<unsigned long long> eout;     // kernel-sorted evicted keys: full | masked
    int64_t last_sel[4] = {0, 0, 0, 0};  // levels, full sweeps, compaction level, candidates
    uint32_t last_window = 0;            // single-sweep window: 0 off, 1 used, 2 estimate missed
    int evict_sample = -1;               // window sample stride: -1 auto, 0 off, S fixed (debug)
    int64_t cand_cap_override = -1;      // test hook (cache_debug_set_evict_cand_cap); -1 = auto
    // distributed fused eviction (cache_evict_sel_*): the kernel arguments across the phases
    SelArgs dsel{};
    int dsel_level = -1;                 // next level expected (-1: none begun)
    bool dsel_push = false;
    bool dsel_done = false;              // the last pick finished the selection
    DevBuf<SelState> dstate;
    DevBuf<uint32_t> dlhist;             // this rank's local level histograms [levels][4096]
    int64_t last_ev_n = 0;               // unit keys of the last eviction (sorted, in ekey), in order
    int64_t last_nd = 0;
    unsigned long long* ev_full = nullptr;   // device: the sorted full keys of the last eviction
    // match predictor (NEXT-3)
    DevBuf<float> pw, prho, pgpart;
    DevBuf<uint32_t> pkeys;
    DevBuf<unsigned int> pcpart, phist;
    DevBuf<EvictState> pst, pst_init;
    cudaStream_t pstream = nullptr;      // private stream of the captured training graph
    cudaEvent_t pev[2] = {nullptr, nullptr};
    bool pred_ok = false;
    // sharding
    int rank = 0, world = 1;
    bool alias = false;   // declared latent aliasing (cache_config.latent_alias)
    PeerPtrs peers{};
    bool peers_ok = false;
    std::vector<void*> ipc_opened;   // peer allocations opened through CUDA IPC
    // push exchange (cache_push_*): this rank's arena and every rank's arena base
    uint8_t* arena = nullptr;
    int64_t arena_nb = 0;
    int32_t arena_topk = 0;
    uint8_t* peer_arena[kMaxWorld] = {};
    bool push_ok = false;
    uint32_t push_epoch = 0;
    int64_t push_nb = -1;
    int push_phase = 0;              // last phase run (1..3), for call-order checks
    uint32_t evict_epoch = 0;        // fused distributed evictions so far
    // failure detection of the push exchange: a peer wait that times out sets the device abort
    // word (consumers skip their peer accesses) and the mapped host word (the host reports
    // CACHE_E_NCCL from then on instead of hanging or trapping)
    DevBuf<uint32_t> abortw;
    uint32_t* errw_h = nullptr;      // pinned, mapped
    uint32_t* errw_d = nullptr;      // its device alias
    unsigned long long peer_timeout_ns = 10ull * 1000 * 1000 * 1000;
    int evict_pass = -1;             // last pass whose pick ran (-1: none / done)
};

static bool peer_failed(const cache_t* c) { return c->errw_h && *(volatile const uint32_t*)c->errw_h != 0u; }

static cache_status peer_fail(const char* where) {
    return fail(CACHE_E_NCCL, std::string(where) + ": a peer rank did not publish within the peer timeout (dead or "
                              "stalled rank); the sharded exchange of this handle is stopped -- rebuild it");
}

extern "C" {

const char* cache_last_error(void) { return g_err.c_str(); }

void cache_default_config(cache_config* cfg) {
    if (!cfg) return;
    std::memset(cfg, 0, sizeof(*cfg));
    cfg->dim = 768;                                    // CLIP text embedding
    cfg->latent_bytes = 4 * 64 * 64 * 2;               // 4x64x64 fp16 latent (BASELINE configs)
    cfg->num_k = 5;                                    // K in {5,10,15,20,25}
    const int kv[5] = {5, 10, 15, 20, 25};
    const double th[5] = {0.65, 0.75, 0.85, 0.90, 0.95};   // Fig. 11
    for (int j = 0; j < 5; ++j) { cfg->k_values[j] = kv[j]; cfg->thresholds[j] = th[j]; }
    cfg->k_bias = 0;
    cfg->max_topk = CACHE_MAX_TOPK;
    cfg->shard_rank = 0;
    cfg->shard_world = 1;
}

// Eviction workspaces for `items` evicted items and `entries` dirty entries (device lists, sort
// scratch, pinned host staging).  Reserved at create for the paper's maintenance rate (1% of
// the stored states per round, C5) so the first evictions do not pay cudaMalloc / pinning
// (measured at 12.5M entries: 46 ms of allocation + 13 ms of pinning in the first call, 2.2 ms
// in steady state); larger evictions still grow them on demand.
static cudaError_t reserve_evict(cache_t* c, int64_t items, int64_t entries) {
    cudaError_t e;
    const size_t pb = (size_t)std::max(items, entries);
    if ((e = c->ekey.ensure_grow(items)) != cudaSuccess) return e;
    if ((e = c->ekey2.ensure_grow(pb)) != cudaSuccess) return e;
    if ((e = c->epool.ensure_grow(items)) != cudaSuccess) return e;
    if ((e = c->eslot.ensure_grow(items)) != cudaSuccess) return e;
    if ((e = c->escr.ensure_grow(sort_scratch_words((int64_t)pb))) != cudaSuccess) return e;
    if ((e = c->edirty.ensure_grow(entries)) != cudaSuccess) return e;
    if ((e = c->edid.ensure_grow(entries)) != cudaSuccess) return e;
    if ((e = c->hev_sorted.ensure(items * 8)) != cudaSuccess) return e;
    if (!c->alias && (e = c->hev_pool.ensure(items * 8)) != cudaSuccess) return e;
    if ((e = c->hev_ds.ensure(entries * 8)) != cudaSuccess) return e;
    // fused eviction: candidate buffers (1/16 of the units) and the per-level histograms
    const int64_t ccap = std::max<int64_t>(65536, c->cap * c->num_k / 16);
    if ((e = c->ckey.ensure_grow(ccap)) != cudaSuccess) return e;
    if ((e = c->cslot.ensure_grow(ccap)) != cudaSuccess) return e;
    if ((e = c->selws.ensure((size_t)(kSelMaxLevels + 1) * kSelBins * 4 + sizeof(SelOut) + 4 * 4096 * 4)) != cudaSuccess)
        return e;
    if ((e = c->ebits.ensure_grow(2 * (c->cap_pad / 32) + (c->alias ? 0 : (c->lcap + 31) / 32) + kEvBitsWords + 1024)) !=
        cudaSuccess)
        return e;
    if ((e = c->eout.ensure_grow(2 * items)) != cudaSuccess) return e;
    return c->hev_did.ensure(entries * 8);
}

cache_status cache_create(const cache_config* cfg, int device, cache_t** out) {
    if (!cfg || !out) return fail(CACHE_E_INVALID_ARG, "cache_create: null argument");
    *out = nullptr;
    if (cfg->dim <= 0 || cfg->dim % 64 != 0 || cfg->dim > kMaxDim)
        return fail(CACHE_E_DIM, "cache_create: dim must be a positive multiple of 64, <= 1024");
    if (cfg->entry_capacity <= 0 || cfg->entry_capacity > 0xFFFFFFFFll || cfg->latent_capacity < 0 ||
        cfg->latent_bytes < 0 || cfg->latent_bytes % 16 != 0)
        return fail(CACHE_E_INVALID_ARG, "cache_create: bad capacity / latent_bytes (multiple of 16)");
    if (cfg->num_k <= 0 || cfg->num_k > CACHE_MAX_K || cfg->k_bias < 0 || cfg->max_topk <= 0 ||
        cfg->max_topk > CACHE_MAX_TOPK)
        return fail(CACHE_E_INVALID_ARG, "cache_create: bad num_k / k_bias / max_topk");
    if (cfg->k_values[0] <= 0) return fail(CACHE_E_INVALID_ARG, "cache_create: K values must be > 0");
    for (int j = 1; j < cfg->num_k; ++j)
        if (cfg->k_values[j] <= cfg->k_values[j - 1] || !(cfg->thresholds[j] >= cfg->thresholds[j - 1]))
            return fail(CACHE_E_INVALID_ARG,
                        "cache_create: K values must increase and thresholds must not decrease (R6)");
    if (cfg->shard_world < 1 || cfg->shard_world > kMaxWorld || cfg->shard_rank < 0 ||
        cfg->shard_rank >= cfg->shard_world)
        return fail(CACHE_E_INVALID_ARG, "cache_create: bad shard_rank / shard_world (world <= 16)");
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(CACHE_E_INVALID_ARG, "cache_create: bad device");
    DeviceGuard g(device);
    cache_t* c = new cache_t();
    c->cfg = *cfg;
    c->device = device;
    c->dim = cfg->dim;
    c->num_k = cfg->num_k;
    c->cap = cfg->entry_capacity;
    c->cap_pad = (cfg->entry_capacity + kTileN - 1) / kTileN * kTileN;
    c->lcap = cfg->latent_capacity;
    c->L = cfg->latent_bytes;
    for (int j = 0; j < c->num_k; ++j) { c->km.thr[j] = cfg->thresholds[j]; c->km.kv[j] = cfg->k_values[j]; }
    c->km.num_k = c->num_k;
    c->km.k_bias = cfg->k_bias;
    c->km.policy = cfg->evict_policy;
    c->km.gran = cfg->evict_granularity;
    if (cfg->evict_granularity != CACHE_EVICT_ITEM && cfg->evict_granularity != CACHE_EVICT_ENTRY) {
        delete c;
        return fail(CACHE_E_INVALID_ARG, "cache_create: bad evict_granularity");
    }
    if (cfg->evict_policy < CACHE_POLICY_LCBFU || cfg->evict_policy > CACHE_POLICY_FIFO) {
        delete c;
        return fail(CACHE_E_INVALID_ARG, "cache_create: bad evict_policy");
    }
    c->rank = cfg->shard_rank;
    c->world = cfg->shard_world;
    c->alias = cfg->latent_alias != 0;
    if (c->alias && c->lcap <= 0) {
        delete c;
        return fail(CACHE_E_INVALID_ARG, "cache_create: latent_alias needs latent_capacity > 0");
    }
    cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
    auto bail = [&](cudaError_t e, const char* what) {
        cache_destroy(c);
        return fail(e == cudaErrorMemoryAllocation ? CACHE_E_OOM : CACHE_E_CUDA,
                    std::string("cache_create: ") + what + ": " + cudaGetErrorString(e));
    };
    cudaError_t e;
    if ((e = cudaMalloc(&c->emb, (size_t)c->cap_pad * c->dim * 2)) != cudaSuccess) return bail(e, "emb");
    if ((e = cudaMalloc(&c->inv_e, (size_t)c->cap_pad * 4)) != cudaSuccess) return bail(e, "inv_e");
    if ((e = cudaMalloc(&c->ids, (size_t)c->cap_pad * 4)) != cudaSuccess) return bail(e, "ids");
    if ((e = cudaMalloc(&c->present, (size_t)c->cap_pad * 4)) != cudaSuccess) return bail(e, "present");
    if ((e = cudaMalloc(&c->lslot, (size_t)c->cap_pad * c->num_k * 4)) != cudaSuccess) return bail(e, "lslot");
    if ((e = cudaMalloc(&c->fcnt, (size_t)c->cap_pad * c->num_k * 4)) != cudaSuccess) return bail(e, "f");
    if ((e = cudaMalloc(&c->lastacc, (size_t)c->cap_pad * c->num_k * 4)) != cudaSuccess) return bail(e, "lastacc");
    if (c->lcap > 0 && c->L > 0 && (e = cudaMalloc(&c->pool, (size_t)c->lcap * c->L)) != cudaSuccess)
        return bail(e, "latent pool");
    cudaMemset(c->emb, 0, (size_t)c->cap_pad * c->dim * 2);
    cudaMemset(c->inv_e, 0xFF, (size_t)c->cap_pad * 4);   // 0xFFFFFFFF = NaN: empty slot
    cudaMemset(c->ids, 0, (size_t)c->cap_pad * 4);
    cudaMemset(c->present, 0, (size_t)c->cap_pad * 4);
    cudaMemset(c->lslot, 0xFF, (size_t)c->cap_pad * c->num_k * 4);
    cudaMemset(c->fcnt, 0, (size_t)c->cap_pad * c->num_k * 4);
    cudaMemset(c->lastacc, 0, (size_t)c->cap_pad * c->num_k * 4);
    if ((e = c->abortw.ensure(1)) != cudaSuccess) return bail(e, "abort word");
    cudaMemset(c->abortw.p, 0, 4);
    if ((e = cudaHostAlloc((void**)&c->errw_h, 64, cudaHostAllocMapped)) != cudaSuccess) return bail(e, "error word");
    *(volatile uint32_t*)c->errw_h = 0u;
    if ((e = cudaHostGetDevicePointer((void**)&c->errw_d, c->errw_h, 0)) != cudaSuccess) return bail(e, "error word");
    if (const char* t = std::getenv("NIRVANA_PEER_TIMEOUT_MS")) c->peer_timeout_ns = std::strtoull(t, nullptr, 10) * 1000000ull;
    if ((e = cudaDeviceSynchronize()) != cudaSuccess) return bail(e, "init");
    c->tm_e_ok = encode_rows(&c->tm_e, c->emb, c->cap_pad, c->dim, 256) &&
                 encode_rows(&c->tm_e128, c->emb, c->cap_pad, c->dim, 128);
    c->h_live.assign(c->cap_pad, 0);
    c->h_ids.assign(c->cap_pad, 0);
    c->free_e.resize(c->cap);
    for (int64_t i = 0; i < c->cap; ++i) c->free_e[i] = c->cap - 1 - i;
    c->free_l.resize(c->lcap);
    for (int64_t i = 0; i < c->lcap; ++i) c->free_l[i] = c->lcap - 1 - i;
    // best effort: without the reservation the workspaces are simply allocated on demand
    if (reserve_evict(c, std::max<int64_t>(4096, c->cap * c->num_k / 100), std::max<int64_t>(1024, c->cap / 100)) !=
        cudaSuccess)
        cudaGetLastError();
    *out = c;
    return CACHE_OK;
}

cache_status cache_destroy(cache_t* c) {
    if (!c) return CACHE_OK;
    DeviceGuard g(c->device);
    cudaDeviceSynchronize();
    for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
    if (c->h_out) cudaFreeHost(c->h_out);
    for (auto& a : c->aslot) {
        a.in.release();
        a.out.release();
        if (a.h_out) cudaFreeHost(a.h_out);
        for (cudaEvent_t e : {a.copied, a.consumed, a.done})
            if (e) cudaEventDestroy(e);
    }
    for (cudaEvent_t e : c->hev)
        if (e) cudaEventDestroy(e);
    if (c->ev_first) cudaEventDestroy(c->ev_first);
    if (c->hcopy) cudaStreamDestroy(c->hcopy);
    if (c->pstream) cudaStreamDestroy(c->pstream);
    for (cudaEvent_t e : c->pev)
        if (e) cudaEventDestroy(e);
    c->pst_init.release();
    for (cudaEvent_t e : c->qev)
        if (e) cudaEventDestroy(e);
    if (c->qside) cudaStreamDestroy(c->qside);
    c->hq_out.release();
    cudaFree(c->emb); cudaFree(c->inv_e); cudaFree(c->ids); cudaFree(c->present);
    cudaFree(c->lslot); cudaFree(c->fcnt); cudaFree(c->lastacc); cudaFree(c->pool);
    if (c->arena) cudaFree(c->arena);
    c->qbuf.release(); c->ystage.release(); c->invq.release(); c->invstage.release();
    c->qstat.release(); c->istat.release(); c->gk.release(); c->recs.release(); c->iplan.release(); c->cplan.release();
    c->hq_in.release(); c->hq_lat.release();
    c->est.release(); c->ehist.release(); c->ekey.release(); c->ecnt.release();
    c->ekey2.release(); c->eslot.release(); c->escr.release();
    c->hev_sorted.release(); c->hev_pool.release(); c->hev_ds.release();
    c->hev_did.release();
    c->epool.release(); c->edirty.release(); c->edid.release();
    c->ckey.release(); c->cslot.release(); c->selws.release(); c->ebits.release(); c->eout.release();
    c->dstate.release(); c->dlhist.release();
    c->abortw.release();
    if (c->errw_h) cudaFreeHost(c->errw_h);
    delete c;
    return CACHE_OK;
}

cache_status cache_insert(cache_t* c, int64_t n, const void* emb, int32_t emb_dtype, const void* latents,
                          const uint8_t* present, uint64_t* out_ids, int32_t* row_status, void* stream) {
    NvtxScope nvtx_scope_("cache_insert");
    if (!c) return fail(CACHE_E_INVALID_ARG, "cache_insert: null cache");
    if (n < 0 || (n > 0 && !emb) || (emb_dtype != CACHE_DTYPE_F32 && emb_dtype != CACHE_DTYPE_BF16))
        return fail(CACHE_E_INVALID_ARG, "cache_insert: bad n / emb / dtype");
    if (n == 0) return CACHE_OK;
    if (latents && !c->pool) return fail(CACHE_E_INVALID_ARG, "cache_insert: latents given but no pool");
    if (latents && c->alias)
        return fail(CACHE_E_INVALID_ARG, "cache_insert: an aliased pool takes no payload (use cache_pool_write)");
    DeviceGuard g(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    const uint32_t full = (1u << c->num_k) - 1u;
    std::vector<uint8_t> masks(n, (uint8_t)full);
    if (present) CK(cudaMemcpy(masks.data(), present, n, cudaMemcpyDefault));
    const size_t esz = emb_dtype == CACHE_DTYPE_BF16 ? 2 : 4;
    const int64_t chunk = std::min<int64_t>(n, 65536);
    CK(c->ystage.ensure((size_t)chunk * c->dim));
    CK(c->invstage.ensure(chunk));
    CK(c->istat.ensure(chunk));
    std::vector<int32_t> st(n);
    // Statuses first (rejected rows get no id / slot), then the all-or-nothing capacity check.
    int64_t n_valid = 0, n_items = 0;
    for (int64_t off = 0; off < n; off += chunk) {
        const int64_t m = std::min(chunk, n - off);
        launch_normalise((const char*)emb + off * c->dim * esz, emb_dtype, m, c->dim, c->ystage.p,
                         c->invstage.p, c->istat.p, s);
        c->launches++;
        CK(cudaMemcpyAsync(st.data() + off, c->istat.p, m * 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    }
    // Accepted rows get consecutive global ids; with sharding this rank keeps id % world == rank.
    int64_t n_accepted = 0;
    for (int64_t r = 0; r < n; ++r) {
        if (st[r] == CACHE_ROW_OK && (masks[r] & full) == 0) st[r] = CACHE_ROW_NO_ITEMS;
        if (st[r] != CACHE_ROW_OK) continue;
        const uint64_t id = c->next_id + n_accepted++;
        if ((int64_t)(id % (uint64_t)c->world) != c->rank) continue;
        n_valid++;
        n_items += __builtin_popcount(masks[r] & full);
    }
    if (n_valid > (int64_t)c->free_e.size() || (!c->alias && n_items > (int64_t)c->free_l.size()))
        return fail(CACHE_E_FULL, "cache_insert: insufficient entry or latent capacity (evict first)");
    if ((uint64_t)c->next_id + n_accepted > 0xFFFFFFFFull)
        return fail(CACHE_E_STATE, "cache_insert: 32-bit id space exhausted");
    std::vector<InsertPlan> plan;
    std::vector<CopyPlan> cp;
    for (int64_t off = 0; off < n; off += chunk) {
        const int64_t m = std::min(chunk, n - off);
        if (off > 0 || n > chunk) {   // staging holds the last chunk: normalise this one again
            launch_normalise((const char*)emb + off * c->dim * esz, emb_dtype, m, c->dim, c->ystage.p,
                             c->invstage.p, c->istat.p, s);
            c->launches++;
        }
        plan.clear();
        cp.clear();
        for (int64_t r = 0; r < m; ++r) {
            const int64_t gr = off + r;
            if (st[gr] != CACHE_ROW_OK) {
                if (out_ids) out_ids[gr] = CACHE_NO_ID;
                continue;
            }
            InsertPlan p;
            p.id = (uint32_t)c->next_id++;
            if (out_ids) out_ids[gr] = p.id;
            if ((int64_t)(p.id % (uint32_t)c->world) != c->rank) continue;   // another shard's row
            p.src_row = r;
            p.slot = c->free_e.back();
            c->free_e.pop_back();
            p.mask = masks[gr] & full;
            for (int j = 0; j < CACHE_MAX_K; ++j) p.lslot[j] = -1;
            for (int j = 0; j < c->num_k; ++j) {
                if (!((p.mask >> j) & 1u)) continue;
                if (c->alias) {
                    p.lslot[j] = (int32_t)CACHE_ALIAS_SLOT(p.id, j, c->lcap);
                    continue;
                }
                p.lslot[j] = (int32_t)c->free_l.back();
                c->free_l.pop_back();
                if (latents) cp.push_back(CopyPlan{gr * c->num_k + j, p.lslot[j]});
            }
            plan.push_back(p);
            c->h_live[p.slot] = 1;
            c->h_ids[p.slot] = p.id;
            c->hwm = std::max(c->hwm, p.slot + 1);
            c->live_entries++;
            c->live_items += __builtin_popcount(p.mask);
        }
        CK(c->iplan.ensure(std::max<size_t>(plan.size(), 1)));
        CK(cudaMemcpyAsync(c->iplan.p, plan.data(), plan.size() * sizeof(InsertPlan), cudaMemcpyHostToDevice, s));
        launch_insert_commit(c->ystage.p, c->invstage.p, c->iplan.p, (int64_t)plan.size(), c->dim, c->num_k,
                             c->emb, c->inv_e, c->ids, c->present, c->lslot, c->fcnt, c->lastacc, c->clock, s);
        c->launches++;
        if (!cp.empty()) {
            CK(c->cplan.ensure(cp.size()));
            CK(cudaMemcpyAsync(c->cplan.p, cp.data(), cp.size() * sizeof(CopyPlan), cudaMemcpyHostToDevice, s));
            launch_copy_latents((const uint8_t*)latents, c->cplan.p, (int64_t)cp.size(), c->L, c->pool, s);
            c->launches++;
        }
        CK(cudaStreamSynchronize(s));   // plans are host vectors reused by the next chunk
        CK(cudaGetLastError());
    }
    if (row_status) std::memcpy(row_status, st.data(), n * 4);
    return n_accepted == n ? CACHE_OK : fail(CACHE_E_BAD_ROWS, "cache_insert: some rows rejected (row_status)");
}

// Scan of this cache's entries for b normalised query rows qrows (bf16, allocation padded to
// a multiple of 128 rows; gk = the rows' k-th-best gate words, already zeroed): partial top-k
// record lists in c->recs ([parts][b][kmax]); *parts_out = lists per query (0: empty cache).
// recs_at != nullptr: write the lists there (the caller sized it, see query_sliced) and
// record no profiling events.
static cache_status scan_rows(cache_t* c, int64_t b, __nv_bfloat16* qrows, uint32_t* gk, int kmax, cudaStream_t s,
                              int* parts_out, Rec* recs_at = nullptr, bool pad_zeroed = false) {
    const int64_t bpad = (b + 127) / 128 * 128;
    const int64_t n_slots = c->hwm;
    int parts = 0;
    const bool prof_on = c->prof_on && recs_at == nullptr;
    bool prof1 = false;   // prof[1] is recorded right before the scoring launch (after host planning)
    if (n_slots > 0) {
        bool use_tc = false;
        TcPlan tp{};
        if (c->scorer != CACHE_SCORER_STREAM && c->tm_e_ok && tc_supported(c->dim)) {
            // measured (round 1): the tcgen05 scan is at 97-98% of HBM bandwidth for every
            // b <= 128 on 1M entries and tensor-bound above, so AUTO always takes it
            use_tc = true;
        }
        if ((c->scorer == CACHE_SCORER_TC || c->scorer == CACHE_SCORER_TC_SINGLE) && !use_tc)
            return fail(CACHE_E_UNSUPPORTED, "query: tensor-core scorer unavailable for this configuration");
        if (use_tc) {
            // more than one 128-query tile: the CTA-pair kernel (half the operand traffic per SM)
            const bool pair = b > 128 && c->scorer != CACHE_SCORER_TC_SINGLE;
            tp = tc_plan(b, n_slots, c->sm_count, pair);
            parts = tp.parts;
            // (scan_core zeroes the pad rows before the ingest launch instead: a memset between the
            // ingest and the scan would break their programmatic-dependent-launch overlap)
            if (bpad > b && !pad_zeroed) CK(cudaMemsetAsync(qrows + b * c->dim, 0, (bpad - b) * c->dim * 2, s));
            CUtensorMap tm_q;
            if (!encode_rows(&tm_q, qrows, bpad, c->dim, 128))
                return fail(CACHE_E_CUDA, "query: cuTensorMapEncodeTiled failed");
            if (!recs_at) CK(c->recs.ensure((size_t)parts * b * kmax));
            if (prof_on) { CK(cudaEventRecord(c->prof[1], s)); prof1 = true; }
            if (!launch_score_tc(kmax, tp, &tm_q, pair ? &c->tm_e128 : &c->tm_e, c->inv_e, c->ids, c->dim, b,
                                 recs_at ? recs_at : c->recs.p, gk, s))
                return fail(CACHE_E_UNSUPPORTED, "query: tensor-core scorer not built");
            c->launches++;
        } else {
            parts = stream_parts(n_slots, b);
            if (!recs_at) CK(c->recs.ensure((size_t)parts * b * kmax));
            if (prof_on) { CK(cudaEventRecord(c->prof[1], s)); prof1 = true; }
            launch_score_stream(kmax, c->emb, c->inv_e, c->ids, n_slots, c->dim, qrows, b,
                                recs_at ? recs_at : c->recs.p, parts, s);
            c->launches++;
        }
    }
    if (prof_on && !prof1) CK(cudaEventRecord(c->prof[1], s));
    if (prof_on) CK(cudaEventRecord(c->prof[2], s));   // end of the scan
    *parts_out = parts;
    return CACHE_OK;
}

// Query ingest + scan of this cache's entries (scan_rows on c->qbuf).
static cache_status scan_core(cache_t* c, int64_t b, const void* queries, int32_t q_dtype, int kmax,
                              cudaStream_t s, int* parts_out) {
    const int64_t bpad = (b + 127) / 128 * 128;
    CK(c->qbuf.ensure((size_t)bpad * c->dim));
    CK(c->invq.ensure(bpad));
    CK(c->qstat.ensure(bpad));
    CK(c->gk.ensure(bpad));
    if (bpad > b) CK(cudaMemsetAsync(c->qbuf.p + b * c->dim, 0, (bpad - b) * c->dim * 2, s));   // tile padding
    if (c->prof_on) CK(cudaEventRecord(c->prof[0], s));
    launch_normalise(queries, q_dtype, b, c->dim, c->qbuf.p, c->invq.p, c->qstat.p, s, c->gk.p);
    c->launches++;
    return scan_rows(c, b, c->qbuf.p, c->gk.p, kmax, s, parts_out, nullptr, true);
}

// Number of device query slices for a batch of b (1 = one scan launch).
static int query_slices(const cache_t* c, int64_t b) {
    if (c->hwm <= 0 || c->scorer == CACHE_SCORER_STREAM || c->scorer == CACHE_SCORER_TC_SINGLE ||
        !c->tm_e_ok || !tc_supported(c->dim))
        return 1;
    if (c->qslices == 1) return 1;
    if (c->qslices == 0 && b < kDevSplitMin) return 1;
    const int ns = c->qslices > 0 ? c->qslices : kDevSplitAuto;
    const int64_t sub = ((b + ns - 1) / ns + 255) / 256 * 256;
    return (int)((b + sub - 1) / sub);
}

// Large tensor-core batches: one ingest launch, then the scan as ns launches over query
// slices of `sub` rows (multiples of 256), and slice i's finalize + gather -- HBM-bound --
// on a side stream while slice i+1's scan -- tensor-bound -- runs.  One finalize CTA (40
// registers x 256 threads, 160 B of shared memory) fits beside the scan CTA on every SM
// (134 x 384 registers, 221 KiB), so the gather of slice i is hidden behind the next scan;
// only the last slice's finalize is exposed.  Results are identical to one launch: each
// query's answer depends only on its own row and the pre-batch state (R9), the counter
// increments are atomics, and the whole batch is one LRU clock tick.
static cache_status query_sliced(cache_t* c, int64_t b, int ns, const void* queries, int32_t q_dtype,
                                 int32_t topk, int kmax, uint64_t* out_ids, float* out_scores, int32_t* out_k,
                                 void* latent_out, void** out_ptr, int32_t* row_status, cudaStream_t s,
                                 bool tick) {
    const int64_t sub = ((b + ns - 1) / ns + 255) / 256 * 256;
    const int64_t bpad = (b + 127) / 128 * 128;
    CK(c->qbuf.ensure((size_t)bpad * c->dim));
    CK(c->invq.ensure(bpad));
    CK(c->qstat.ensure(bpad));
    CK(c->gk.ensure(bpad));
    int64_t off[kDevSplitMax + 1], roff[kDevSplitMax];
    int parts[kDevSplitMax];
    size_t tot = 0;
    int n = 0;
    for (int64_t o = 0; o < b; o += sub, ++n) {
        const int64_t nb = std::min(sub, b - o);
        off[n] = o;
        parts[n] = tc_plan(nb, c->hwm, c->sm_count, nb > 128).parts;
        roff[n] = (int64_t)tot;
        tot += (size_t)parts[n] * nb * kmax;
    }
    off[n] = b;
    if (n != ns) return fail(CACHE_E_STATE, "query: slice plan mismatch");
    CK(c->recs.ensure(tot));   // before any launch: the buffer is not reallocated under a slice
    if (!c->qside) CK(cudaStreamCreateWithFlags(&c->qside, cudaStreamNonBlocking));
    for (cudaEvent_t& e : c->qev)
        if (!e) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    if (c->prof_on) CK(cudaEventRecord(c->prof[0], s));
    launch_normalise(queries, q_dtype, b, c->dim, c->qbuf.p, c->invq.p, c->qstat.p, s, c->gk.p);
    c->launches++;
    if (c->prof_on) CK(cudaEventRecord(c->prof[1], s));
    for (int i = 0; i < n; ++i) {
        const int64_t nb = off[i + 1] - off[i];
        int p = 0;
        cache_status r = scan_rows(c, nb, c->qbuf.p + off[i] * c->dim, c->gk.p + off[i], kmax, s, &p,
                                   c->recs.p + roff[i]);
        if (r != CACHE_OK) return r;
        if (p != parts[i]) return fail(CACHE_E_STATE, "query: slice parts mismatch");
        if (i + 1 < n) CK(cudaEventRecord(c->qev[i], s));
    }
    if (c->prof_on) CK(cudaEventRecord(c->prof[2], s));
    if (tick) c->clock++;   // one query batch = one tick of the LRU clock
    uint8_t* lat = (uint8_t*)latent_out;
    for (int i = 0; i < n; ++i) {
        const int64_t o = off[i], nb = off[i + 1] - off[i];
        const bool last = i + 1 == n;
        cudaStream_t fs = last ? s : c->qside;
        if (!last) CK(cudaStreamWaitEvent(c->qside, c->qev[i], 0));
        launch_finalize(kmax, c->recs.p + roff[i], parts[i], nb, topk, c->invq.p + o, c->qstat.p + o, c->ids,
                        c->present, c->lslot, c->fcnt, c->lastacc, c->clock, c->pool, c->L, c->km,
                        out_ids + o * topk, out_scores + o * topk, out_k + o, lat ? lat + o * c->L : nullptr,
                        out_ptr ? out_ptr + o : nullptr, row_status ? row_status + o : nullptr, fs, last);
        c->launches++;
    }
    if (c->prof_on) CK(cudaEventRecord(c->prof[3], s));
    CK(cudaEventRecord(c->qev[kDevSplitMax], c->qside));   // join: s continues after every slice
    CK(cudaStreamWaitEvent(s, c->qev[kDevSplitMax], 0));
    CK(cudaGetLastError());
    c->queries += b;
    return CACHE_OK;
}

// tick = false: a later sub-batch of the same host batch (same LRU clock value).
static cache_status query_core(cache_t* c, int64_t b, const void* queries, int32_t q_dtype, int32_t topk,
                               uint64_t* out_ids, float* out_scores, int32_t* out_k, void* latent_out,
                               void** out_ptr, int32_t* row_status, cudaStream_t s, bool tick = true,
                               bool count = true) {
    const int kmax = topk == 1 ? 1 : (topk <= 4 ? 4 : 16);
    const int ns = query_slices(c, b);
    if (ns > 1 && count)
        return query_sliced(c, b, ns, queries, q_dtype, topk, kmax, out_ids, out_scores, out_k, latent_out, out_ptr,
                            row_status, s, tick);
    int parts = 0;
    cache_status r = scan_core(c, b, queries, q_dtype, kmax, s, &parts);
    if (r != CACHE_OK) return r;
    if (c->prof_on) CK(cudaEventRecord(c->prof[2], s));
    if (tick) c->clock++;   // one query batch = one tick of the LRU clock
    launch_finalize(kmax, c->recs.p, parts, b, topk, c->invq.p, c->qstat.p, c->ids, c->present, c->lslot,
                    count ? c->fcnt : nullptr, count ? c->lastacc : nullptr, c->clock, c->pool, c->L, c->km, out_ids, out_scores, out_k,
                    (uint8_t*)latent_out, out_ptr, row_status, s);
    c->launches++;
    if (c->prof_on) CK(cudaEventRecord(c->prof[3], s));
    CK(cudaGetLastError());
    if (count) c->queries += b;
    return CACHE_OK;
}

cache_status cache_query_batch(cache_t* c, int64_t b, const void* queries, int32_t q_dtype, int32_t topk,
                               uint64_t* out_ids, float* out_scores, int32_t* out_k, void* latent_out,
                               void** out_latent_ptr, int32_t* row_status, void* stream) {
    NvtxScope nvtx_scope_("cache_query_batch");
    if (!c) return fail(CACHE_E_INVALID_ARG, "cache_query_batch: null cache");
    if (b < 0 || b > 0x7FFFFFFF || topk < 1 || topk > c->cfg.max_topk ||
        (q_dtype != CACHE_DTYPE_F32 && q_dtype != CACHE_DTYPE_BF16))
        return fail(CACHE_E_INVALID_ARG, "cache_query_batch: bad b / topk / dtype");
    if (b == 0) return CACHE_OK;
    if (!queries || !out_ids || !out_scores || !out_k)
        return fail(CACHE_E_INVALID_ARG, "cache_query_batch: null buffer");
    if (latent_out && !c->pool) return fail(CACHE_E_INVALID_ARG, "cache_query_batch: no latent pool");
    DeviceGuard g(c->device);
    return query_core(c, b, queries, q_dtype, topk, out_ids, out_scores, out_k, latent_out, out_latent_ptr,
                      row_status, (cudaStream_t)stream);
}

cache_status cache_query_peek(cache_t* c, int64_t b, const void* queries, int32_t q_dtype, int32_t topk,
                              uint64_t* out_ids, float* out_scores, int32_t* out_k, int32_t* row_status,
                              void* stream) {
    NvtxScope nvtx_scope_("cache_query_peek");
    if (!c) return fail(CACHE_E_INVALID_ARG, "cache_query_peek: null cache");
    if (b < 0 || b > 0x7FFFFFFF || topk < 1 || topk > c->cfg.max_topk ||
        (q_dtype != CACHE_DTYPE_F32 && q_dtype != CACHE_DTYPE_BF16))
        return fail(CACHE_E_INVALID_ARG, "cache_query_peek: bad b / topk / dtype");
    if (b == 0) return CACHE_OK;
    if (!queries || !out_ids || !out_scores || !out_k) return fail(CACHE_E_INVALID_ARG, "cache_query_peek: null buffer");
    DeviceGuard g(c->device);
    return query_core(c, b, queries, q_dtype, topk, out_ids, out_scores, out_k, nullptr, nullptr, row_status,
                      (cudaStream_t)stream, /*tick=*/false, /*count=*/false);
}

cache_status cache_query_local(cache_t* c, int64_t b, const void* queries, int32_t q_dtype, int32_t topk,
                               cache_shard_rec* out_recs, void* stream) {
    NvtxScope nvtx_scope_("cache_query_local");
    if (!c) return fail(CACHE_E_INVALID_ARG, "cache_query_local: null cache");
    if (b < 0 || b > 0x7FFFFFFF || topk < 1 || topk > c->cfg.max_topk ||
        (q_dtype != CACHE_DTYPE_F32 && q_dtype != CACHE_DTYPE_BF16))
        return fail(CACHE_E_INVALID_ARG, "cache_query_local: bad b / topk / dtype");
    if (b == 0) return CACHE_OK;
    if (!queries || !out_recs) return fail(CACHE_E_INVALID_ARG, "cache_query_local: null buffer");
    DeviceGuard g(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    const int kmax = topk == 1 ? 1 : (topk <= 4 ? 4 : 16);
    int parts = 0;
    cache_status r = scan_core(c, b, queries, q_dtype, kmax, s, &parts);
    if (r != CACHE_OK) return r;
    launch_local_merge(kmax, c->recs.p, parts, b, topk, c->qstat.p, c->present, c->rank, out_recs, s);
    c->launches++;
    CK(cudaGetLastError());
    return CACHE_OK;
}

cache_status cache_query_merge(cache_t* c, int64_t b, int64_t row0, int64_t nb, int32_t topk,
                               const cache_shard_rec* recs, uint64_t* out_ids, float* out_scores, int32_t* out_k,
                               void* latent_out, void** out_latent_ptr, int32_t* row_status, void* stream) {
    NvtxScope nvtx_scope_("cache_query_merge");
    if (!c) return fail(CACHE_E_INVALID_ARG, "cache_query_merge: null cache");
    if (b < 0 || row0 < 0 || nb < 0 || row0 + nb > b || topk < 1 || topk > c->cfg.max_topk)
        return fail(CACHE_E_INVALID_ARG, "cache_query_merge: bad b / row range / topk");
    if (nb == 0) return CACHE_OK;
    if (!recs || !out_ids || !out_scores || !out_k) return fail(CACHE_E_INVALID_ARG, "cache_query_merge: null buffer");
    if (!c->peers_ok) return fail(CACHE_E_STATE, "cache_query_merge: cache_attach_peers not called");
    if (c->qstat.n < (size_t)b) return fail(CACHE_E_STATE, "cache_query_merge: no matching cache_query_local batch");
    DeviceGuard g(c->device);
    const int kmax = topk == 1 ? 1 : (topk <= 4 ? 4 : 16);
    c->clock++;   // every rank merges once per global batch -> the clocks agree across ranks
    launch_merge_sharded(kmax, recs, b, row0, c->world, row0, nb, topk, c->invq.p, c->qstat.p, c->peers, c->clock,
                         c->L, c->km, out_ids, out_scores, out_k, (uint8_t*)latent_out, out_latent_ptr, row_status,
                         (cudaStream_t)stream);
    c->launches++;
    CK(cudaGetLastError());
    c->queries += nb;
    return CACHE_OK;
}

// ---- cache-selector profiling (Alg. 2) ----
cache_status cache_profile_thresholds(cache_t* c, int64_t b, const void* queries, int32_t q_dtype, const float* quality,
                                      double alpha, double* out_thresholds, int64_t* out_failed, void* stream) {
    NvtxScope nvtx_scope_("cache_profile_thresholds");
    if (!c) return fail(CACHE_E_INVALID_ARG, "cache_profile_thresholds: null cache");
    if (b <= 0 || b > 0x7FFFFFFF || !queries || !quality || !out_thresholds ||
        (q_dtype != CACHE_DTYPE_F32 && q_dtype != CACHE_DTYPE_BF16) || !(alpha == alpha))
        return fail(CACHE_E_INVALID_ARG, "cache_profile_thresholds: bad argument");
    if (c->live_entries == 0) return fail(CACHE_E_STATE, "cache_profile_thresholds: empty cache");
    DeviceGuard g(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    int parts = 0;
    cache_status r = scan_core(c, b, queries, q_dtype, 1, s, &parts);   // exact top-1, no access counted
    if (r != CACHE_OK) return r;
    DevBuf<cache_shard_rec> recs;
    DevBuf<uint32_t> red;   // fail[num_k] | smin
    CK(recs.ensure(b));
    CK(red.ensure(c->num_k + 1));
    CK(cudaMemsetAsync(red.p, 0, c->num_k * 4, s));
    CK(cudaMemsetAsync(red.p + c->num_k, 0xFF, 4, s));
    launch_local_merge(1, c->recs.p, parts, b, 1, c->qstat.p, c->present, c->rank, recs.p, s);
    launch_profile_reduce(recs.p, c->invq.p, c->qstat.p, b, quality, c->num_k, (float)alpha, red.p, red.p + c->num_k, s);
    c->launches += 2;
    std::vector<uint32_t> h(c->num_k + 1);
    CK(cudaMemcpyAsync(h.data(), red.p, (c->num_k + 1) * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    recs.release();
    red.release();
    auto from_orderable = [](uint32_t o) {
        const uint32_t u = (o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o;
        float f;
        std::memcpy(&f, &u, 4);
        return (double)f;
    };
    if (h[c->num_k] == 0xFFFFFFFFu) return fail(CACHE_E_STATE, "cache_profile_thresholds: no profiling query had a valid match");
    const double smin = from_orderable(h[c->num_k]);
    double prev = -INFINITY;
    for (int j = 0; j < c->num_k; ++j) {
        // R25: no failing pair -> the smallest profiled similarity (the evidence's lower edge);
        // thresholds made non-decreasing in K (a larger K never applies below a smaller one's)
        double t = h[j] ? from_orderable(h[j]) : smin;
        if (out_failed) out_failed[j] = h[j] ? 1 : 0;
        t = std::max(t, prev);
        out_thresholds[j] = prev = t;
    }
    return CACHE_OK;
}

cache_status cache_set_thresholds(cache_t* c, const double* thresholds) {
    if (!c || !thresholds) return fail(CACHE_E_INVALID_ARG, "cache_set_thresholds: null argument");
    for (int j = 0; j < c->num_k; ++j)
        if (!(thresholds[j] == thresholds[j]) || (j > 0 && thresholds[j] < thresholds[j - 1]))
            return fail(CACHE_E_INVALID_ARG, "cache_set_thresholds: thresholds must be non-decreasing numbers");
    for (int j = 0; j < c->num_k; ++j) c->km.thr[j] = c->cfg.thresholds[j] = thresholds[j];
    return CACHE_OK;
}

cache_status cache_predictor_train(cache_t* c, double nu, int32_t epochs, double lr0, void* stream) {
    NvtxScope nvtx_scope_("cache_predictor_train");
    if (!c || !(nu > 0.0 && nu < 1.0) || epochs < 0 || !(lr0 > 0.0))
        return fail(CACHE_E_INVALID_ARG, "cache_predictor_train: bad nu / epochs / lr0");
    if (c->live_entries <= 0) return fail(CACHE_E_STATE, "cache_predictor_train: empty cache");
    DeviceGuard g(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t n_slots = c->hwm, n = c->live_entries;
    const int nblk = (int)std::max<int64_t>(1, std::min<int64_t>(296, n_slots));
    CK(c->pw.ensure(c->dim));
    CK(c->prho.ensure(1));
    CK(c->pkeys.ensure(n_slots));
    CK(c->pgpart.ensure((size_t)nblk * c->dim));
    CK(c->pcpart.ensure(nblk));
    CK(c->phist.ensure(256));
    CK(c->pst.ensure(1));
    const unsigned long long k = (unsigned long long)std::max<double>(1.0, std::ceil(nu * (double)n));
    // w0 = mean of the unit-scaled cached embeddings (keys of live rows first, w = 0)
    CK(cudaMemsetAsync(c->pst.p, 0, sizeof(EvictState), s));
    CK(cudaMemsetAsync(c->pw.p, 0, c->dim * 4, s));
    CK(cudaMemsetAsync(c->phist.p, 0, 256 * 4, s));
    pred_margins(c->emb, c->inv_e, n_slots, c->dim, c->pw.p, c->pkeys.p, s);
    pred_viol(c->emb, c->inv_e, c->pkeys.p, n_slots, c->dim, c->pst.p, 1, c->pgpart.p, c->pcpart.p, nblk, s);
    pred_update(c->pgpart.p, c->pcpart.p, nblk, c->dim, c->pw.p, nu, 0.0, n, 0, s);
    c->launches += 3;
    // The epoch loop is 11 dependent launches per epoch.  NIRVANA_PRED_GRAPH=1 captures it into
    // a CUDA graph on a private stream per call: measured 8.3 vs 8.0 ms for 50 epochs at 100K
    // entries (the capture + instantiation cost what the launches cost; the epochs are not
    // launch-bound after all), so the plain launches stay the default.
    static const bool use_graph = [] {
        const char* e = std::getenv("NIRVANA_PRED_GRAPH");
        return e && e[0] == '1';
    }();
    const EvictState st0{0ull, 0ull, k};
    CK(c->pst_init.ensure(1));
    CK(cudaMemcpyAsync(c->pst_init.p, &st0, sizeof(st0), cudaMemcpyHostToDevice, s));
    auto epochs_on = [&](cudaStream_t q) {
        for (int t = 0; t <= epochs; ++t) {
            cudaMemcpyAsync(c->pst.p, c->pst_init.p, sizeof(EvictState), cudaMemcpyDeviceToDevice, q);
            pred_margins(c->emb, c->inv_e, n_slots, c->dim, c->pw.p, c->pkeys.p, q);
            pred_select(c->pkeys.p, n_slots, c->pst.p, c->phist.p, q);   // rho = k-th smallest margin
            if (t == epochs) break;
            pred_viol(c->emb, c->inv_e, c->pkeys.p, n_slots, c->dim, c->pst.p, 0, c->pgpart.p, c->pcpart.p, nblk, q);
            pred_update(c->pgpart.p, c->pcpart.p, nblk, c->dim, c->pw.p, nu, lr0 / std::sqrt(1.0 + t), n, 1, q);
        }
    };
    c->launches += (int64_t)(epochs + 1) * 9 + (int64_t)epochs * 2;
    cudaGraphExec_t pexec = nullptr;
    if (use_graph) {
        if (!c->pstream) CK(cudaStreamCreateWithFlags(&c->pstream, cudaStreamNonBlocking));
        if (!c->pev[0]) {
            CK(cudaEventCreateWithFlags(&c->pev[0], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&c->pev[1], cudaEventDisableTiming));
        }
        CK(cudaEventRecord(c->pev[0], s));
        CK(cudaStreamWaitEvent(c->pstream, c->pev[0], 0));
        cudaGraph_t graph = nullptr;
        CK(cudaStreamBeginCapture(c->pstream, cudaStreamCaptureModeThreadLocal));
        epochs_on(c->pstream);
        CK(cudaStreamEndCapture(c->pstream, &graph));
        cudaError_t e = cudaGraphInstantiate(&pexec, graph, 0);
        cudaGraphDestroy(graph);
        if (e == cudaSuccess) e = cudaGraphLaunch(pexec, c->pstream);
        CK(e);
        CK(cudaEventRecord(c->pev[1], c->pstream));
        CK(cudaStreamWaitEvent(s, c->pev[1], 0));
    } else {
        epochs_on(s);
    }
    pred_finish(c->pst.p, c->prho.p, s);
    c->launches++;
    const cudaError_t se = cudaStreamSynchronize(s);
    if (pexec) cudaGraphExecDestroy(pexec);
    CK(se);
    CK(cudaGetLastError());
    c->pred_ok = true;
    return CACHE_OK;
}

cache_status cache_predict(cache_t* c, int64_t b, const void* queries, int32_t q_dtype, uint8_t* out_flags,
                           float* out_margin, void* stream) {
    NvtxScope nvtx_scope_("cache_predict");
    if (!c || b < 0 || (b > 0 && !queries) || (q_dtype != CACHE_DTYPE_F32 && q_dtype != CACHE_DTYPE_BF16))
        return fail(CACHE_E_INVALID_ARG, "cache_predict: bad argument");
    if (!c->pred_ok) return fail(CACHE_E_STATE, "cache_predict: predictor not trained");
    if (b == 0) return CACHE_OK;
    DeviceGuard g(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t bpad = (b + 127) / 128 * 128;
    CK(c->qbuf.ensure((size_t)bpad * c->dim));
    CK(c->invq.ensure(bpad));
    CK(c->qstat.ensure(bpad));
    launch_normalise(queries, q_dtype, b, c->dim, c->qbuf.p, c->invq.p, c->qstat.p, s);
    pred_predict(c->qbuf.p, c->invq.p, c->qstat.p, b, c->dim, c->pw.p, c->prho.p, out_flags, out_margin, s);
    c->launches += 2;
    CK(cudaGetLastError());
    return CACHE_OK;
}

cache_status cache_predictor_get(cache_t* c, float* w, float* rho) {
    if (!c || !w || !rho) return fail(CACHE_E_INVALID_ARG, "cache_predictor_get: null argument");
    if (!c->pred_ok) return fail(CACHE_E_STATE, "cache_predictor_get: predictor not trained");
    DeviceGuard g(c->device);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(w, c->pw.p, c->dim * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(rho, c->prho.p, 4, cudaMemcpyDeviceToHost));
    return CACHE_OK;
}

cache_status cache_pool_write(cache_t* c, int64_t slot0, int64_t n, const void* src, void* stream) {
    if (!c || slot0 < 0 || n < 0 || slot0 + n > c->lcap || (n > 0 && !src) || !c->pool)
        return fail(CACHE_E_INVALID_ARG, "cache_pool_write: bad slot range / source / no pool");
    if (n == 0) return CACHE_OK;
    DeviceGuard g(c->device);
    CK(cudaMemcpyAsync(c->pool + slot0 * c->L, src, (size_t)n * c->L, cudaMemcpyDefault, (cudaStream_t)stream));
    return CACHE_OK;
}

// Identity of this process for cache_attach_peers: raw device pointers are usable only inside
// the exporting process.  A pid alone is not enough (ranks in separate PID namespaces, e.g. one
// container per GPU, can share one), so every process draws a random 64-bit token once.
static uint64_t process_token() {
    static const uint64_t tok = [] {
        uint64_t t = 0;
        if (FILE* f = std::fopen("/dev/urandom", "rb")) {
            if (std::fread(&t, sizeof(t), 1, f) != 1) t = 0;
            std::fclose(f);
        }
        t ^= (uint64_t)getpid() * 0x9E3779B97F4A7C15ull;
        t ^= (uint64_t)std::chrono::high_resolution_clock::now().time_since_epoch().count();
        return t ? t : 1ull;
    }();
    return tok;
}

cache_status cache_export_peer(cache_t* c, cache_peer_desc* out) {
    if (!c || !out) return fail(CACHE_E_INVALID_ARG, "cache_export_peer: null argument");
    DeviceGuard g(c->device);
    std::memset(out, 0, sizeof(*out));
    out->device = c->device;
    out->pid = (int32_t)getpid();
    out->process_token = process_token();
    out->num_k = c->num_k;
    out->latent_bytes = c->L;
    out->lslot = c->lslot;
    out->fcnt = c->fcnt;
    out->lastacc = c->lastacc;
    out->pool = c->pool;
    cudaIpcMemHandle_t h;
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    CK(cudaIpcGetMemHandle(&h, c->lslot));
    std::memcpy(out->ipc_lslot, &h, 64);
    CK(cudaIpcGetMemHandle(&h, c->fcnt));
    std::memcpy(out->ipc_fcnt, &h, 64);
    CK(cudaIpcGetMemHandle(&h, c->lastacc));
    std::memcpy(out->ipc_lastacc, &h, 64);
    if (c->pool) {
        CK(cudaIpcGetMemHandle(&h, c->pool));
        std::memcpy(out->ipc_pool, &h, 64);
    }
    out->arena = c->arena;
    out->arena_nb = c->arena_nb;
    out->arena_topk = c->arena_topk;
    if (c->arena) {
        CK(cudaIpcGetMemHandle(&h, c->arena));
        std::memcpy(out->ipc_arena, &h, 64);
    }
    return CACHE_OK;
}

cache_status cache_attach_peers(cache_t* c, int32_t world, const cache_peer_desc* descs) {
    if (!c || !descs || world != c->world) return fail(CACHE_E_INVALID_ARG, "cache_attach_peers: bad argument");
    DeviceGuard g(c->device);
    const int32_t me = (int32_t)getpid();
    const uint64_t tok = process_token();
    PeerPtrs p{};
    bool push = c->arena != nullptr;
    uint8_t* pa[kMaxWorld] = {};
    for (int r = 0; r < world; ++r) {
        const cache_peer_desc& d = descs[r];
        if (d.num_k != c->num_k || d.latent_bytes != c->L)
            return fail(CACHE_E_INVALID_ARG, "cache_attach_peers: peer configuration differs");
        if (c->arena && (!d.arena || d.arena_nb != c->arena_nb || d.arena_topk != c->arena_topk))
            push = false;   // some rank has no (or a differently sized) arena: no push exchange
        if (d.pid == me && d.process_token == tok) {   // same process (own rank, or virtual ranks on one GPU)
            p.lslot[r] = (const int32_t*)d.lslot;
            p.fcnt[r] = (uint32_t*)d.fcnt;
            p.lastacc[r] = (uint32_t*)d.lastacc;
            p.pool[r] = (const uint8_t*)d.pool;
            pa[r] = (uint8_t*)d.arena;
            continue;
        }
        if (d.arena && c->arena) {
            void* ap = nullptr;
            cudaIpcMemHandle_t ha;
            std::memcpy(&ha, d.ipc_arena, 64);
            CK(cudaIpcOpenMemHandle(&ap, ha, cudaIpcMemLazyEnablePeerAccess));
            c->ipc_opened.push_back(ap);
            pa[r] = (uint8_t*)ap;
        }
        void* ptr = nullptr;
        cudaIpcMemHandle_t h;
        std::memcpy(&h, d.ipc_lslot, 64);
        CK(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
        c->ipc_opened.push_back(ptr);
        p.lslot[r] = (const int32_t*)ptr;
        std::memcpy(&h, d.ipc_fcnt, 64);
        CK(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
        c->ipc_opened.push_back(ptr);
        p.fcnt[r] = (uint32_t*)ptr;
        std::memcpy(&h, d.ipc_lastacc, 64);
        CK(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
        c->ipc_opened.push_back(ptr);
        p.lastacc[r] = (uint32_t*)ptr;
        if (d.pool) {
            std::memcpy(&h, d.ipc_pool, 64);
            CK(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
            c->ipc_opened.push_back(ptr);
            p.pool[r] = (const uint8_t*)ptr;
        }
    }
    p.abort = c->abortw.p;
    c->peers = p;
    c->peers_ok = true;
    c->push_ok = push;
    for (int r = 0; r < kMaxWorld; ++r) c->peer_arena[r] = r < world ? pa[r] : nullptr;
    return CACHE_OK;
}

cache_status cache_last_evicted_keys(cache_t* c, uint64_t* out, int64_t cap, int64_t* out_n) {
    if (!c || cap < 0 || (cap > 0 && !out)) return fail(CACHE_E_INVALID_ARG, "cache_last_evicted_keys: bad argument");
    const int64_t n = std::min<int64_t>(cap, c->last_ev_n);
    if (n > 0) {   // the sorted full keys stay on the device until the next eviction
        DeviceGuard g(c->device);
        CK(cudaMemcpy(out, c->ev_full ? c->ev_full : c->ekey.p, (size_t)n * 8, cudaMemcpyDeviceToHost));
    }
    if (out_n) *out_n = c->last_ev_n;
    return CACHE_OK;
}

cache_status cache_push_status(cache_t* c, void* stream) {
    if (!c) return fail(CACHE_E_INVALID_ARG, "cache_push_status: null cache");
    DeviceGuard g(c->device);
    CK(cudaStreamSynchronize((cudaStream_t)stream));
    if (peer_failed(c)) return peer_fail("cache_push_status");
    return CACHE_OK;
}

cache_status cache_set_peer_timeout(cache_t* c, int64_t timeout_ms) {
    if (!c || timeout_ms <= 0) return fail(CACHE_E_INVALID_ARG, "cache_set_peer_timeout: bad argument");
    c->peer_timeout_ns = (unsigned long long)timeout_ms * 1000000ull;
    return CACHE_OK;
}

cache_status cache_push_reserve(cache_t* c, int64_t max_nb, int32_t max_topk) {
    if (!c || max_nb < 1 || max_topk < 1 || max_topk > c->cfg.max_topk || (int64_t)c->world * max_nb > 0x7FFFFFFF)
        return fail(CACHE_E_INVALID_ARG, "cache_push_reserve: bad argument");
    if (c->world > kMaxWorld) return fail(CACHE_E_INVALID_ARG, "cache_push_reserve: world too large");
    if (c->peers_ok) return fail(CACHE_E_STATE, "cache_push_reserve: call before cache_export_peer / attach");
    DeviceGuard g(c->device);
    if (c->arena) {
        cudaFree(c->arena);
        c->arena = nullptr;
    }
    const ArenaLayout L = arena_layout(c->world, max_nb, max_topk, c->dim);
    CK(cudaMalloc(&c->arena, L.total));
    CK(cudaMemset(c->arena, 0, L.total));
    CK(cudaDeviceSynchronize());
    c->arena_nb = max_nb;
    c->arena_topk = max_topk;
    c->push_epoch = 0;
    c->push_phase = 0;
    c->evict_epoch = 0;
    c->evict_pass = -1;
    return CACHE_OK;
}

static PushSignal push_signal_of(cache_t* c, size_t flag_off, int counter) {
    PushSignal sg{};
    for (int r = 0; r < c->world; ++r) sg.flag[r] = (uint32_t*)(c->peer_arena[r] + flag_off) + c->rank;
    sg.world = c->world;
    sg.done = (uint32_t*)(c->arena + arena_layout(c->world, c->arena_nb, c->arena_topk, c->dim).done) + counter;
    sg.epoch = c->push_epoch;
    sg.abort = c->abortw.p;
    return sg;
}


static void wait_flags(cache_t* c, const uint32_t* flags, uint32_t epoch, cudaStream_t s) {
    launch_wait_flags(flags, c->world, epoch, c->peer_timeout_ns, c->abortw.p, c->errw_d, s);
}

// ---- fused distributed eviction selection (histograms over peer memory) ----
cache_status cache_push_evict_hist(cache_t* c, int64_t n, int32_t pass, void* stream) {
    if (!c) return fail(CACHE_E_INVALID_ARG, "cache_push_evict_hist: null cache");
    if (peer_failed(c)) return peer_fail("cache_push_evict_hist");
    if (!c->push_ok) return fail(CACHE_E_STATE, "cache_push_evict_hist: no push arenas");
    if (pass < 0 || pass > 7 || (pass == 0 && n < 0)) return fail(CACHE_E_INVALID_ARG, "cache_push_evict_hist: bad pass / n");
    if (pass != c->evict_pass + 1) return fail(CACHE_E_STATE, "cache_push_evict_hist: passes out of order");
    DeviceGuard g(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    const ArenaLayout L = arena_layout(c->world, c->arena_nb, c->arena_topk, c->dim);
    if (pass == 0) {
        CK(c->est.ensure(1));
        EvictState st0{0ull, 0ull, (unsigned long long)n};
        CK(cudaMemcpyAsync(c->est.p, &st0, sizeof(st0), cudaMemcpyHostToDevice, s));
        c->evict_epoch++;
    }
    PushHist ph{};
    for (int r = 0; r < c->world; ++r) ph.dst[r] = (unsigned int*)(c->peer_arena[r] + L.ehist) + 256 * pass;
    ph.world = c->world;
    PushSignal sig = push_signal_of(c, L.eflag + (size_t)pass * kMaxWorld * 4, 2);
    sig.epoch = c->evict_epoch;
    launch_evict_hist_push(c->present, c->fcnt, c->lastacc, c->ids, c->hwm, c->km, c->est.p, pass, ph, sig, s);
    c->launches++;
    CK(cudaGetLastError());
    return CACHE_OK;
}

cache_status cache_push_evict_pick(cache_t* c, int32_t pass, void* stream) {
    if (!c) return fail(CACHE_E_INVALID_ARG, "cache_push_evict_pick: null cache");
    if (peer_failed(c)) return peer_fail("cache_push_evict_pick");
    if (!c->push_ok || pass != c->evict_pass + 1 || pass > 7)
        return fail(CACHE_E_STATE, "cache_push_evict_pick: call after cache_push_evict_hist of the same pass");
    DeviceGuard g(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    const ArenaLayout L = arena_layout(c->world, c->arena_nb, c->arena_topk, c->dim);
    wait_flags(c, (const uint32_t*)(c->arena + L.eflag + (size_t)pass * kMaxWorld * 4), c->evict_epoch, s);
    // the complete global histogram is in this rank's own arena; the pick zeroes it after use
    launch_evict_pick((unsigned int*)(c->arena + L.ehist) + 256 * pass, c->est.p, pass, s);
    c->launches += 2;
    c->evict_pass = pass;
    CK(cudaGetLastError());
    return CACHE_OK;
}

cache_status cache_push_evict_apply(cache_t* c, int64_t n, uint64_t* out_evicted, int64_t* out_n,
                                    uint64_t* out_dirty_ids, int64_t* out_n_dirty, void* stream) {
    if (!c) return fail(CACHE_E_INVALID_ARG, "cache_push_evict_apply: null cache");
    if (peer_failed(c)) return peer_fail("cache_push_evict_apply");
    if (c->evict_pass != 7) return fail(CACHE_E_STATE, "cache_push_evict_apply: the 8 passes have not run");
    c->evict_pass = -1;
    return cache_evict_apply(c, reinterpret_cast<const cache_evict_state*>(c->est.p), n, out_evicted, out_n,
                             out_dirty_ids, out_n_dirty, stream);
}

cache_status cache_push_queries(cache_t* c, int64_t nb, const void* queries, int32_t q_dtype, void* stream) {
    NvtxScope nvtx_scope_("cache_push_queries");
    if (!c) return fail(CACHE_E_INVALID_ARG, "cache_push_queries: null cache");
    if (peer_failed(c)) return peer_fail("cache_push_queries");
    if (!c->push_ok) return fail(CACHE_E_STATE, "cache_push_queries: no push arenas (cache_push_reserve on every rank, then export / attach)");
    if (nb < 0 || nb > c->arena_nb || (nb > 0 && !queries) || (q_dtype != CACHE_DTYPE_F32 && q_dtype != CACHE_DTYPE_BF16))
        return fail(CACHE_E_INVALID_ARG, "cache_push_queries: bad nb / queries / dtype");
    if (c->push_phase != 0 && c->push_phase != 3) return fail(CACHE_E_STATE, "cache_push_queries: previous batch not merged");
    DeviceGuard g(c->device);
    const ArenaLayout L = arena_layout(c->world, c->arena_nb, c->arena_topk, c->dim);
    c->push_epoch++;
    c->push_nb = nb;
    PushRows o{};
    for (int r = 0; r < c->world; ++r) {
        o.y[r] = (__nv_bfloat16*)(c->peer_arena[r] + L.qg);
        o.inv[r] = (float*)(c->peer_arena[r] + L.invq);
        o.status[r] = (int32_t*)(c->peer_arena[r] + L.qstat);
    }
    o.n = c->world;
    launch_normalise_push(queries, q_dtype, nb, c->dim, o, (int64_t)c->rank * nb, push_signal_of(c, L.qflag, 0),
                          (cudaStream_t)stream);
    c->launches++;
    c->push_phase = 1;
    CK(cudaGetLastError());
    return CACHE_OK;
}

cache_status cache_push_scan(cache_t* c, int64_t nb, int32_t topk, void* stream) {
    NvtxScope nvtx_scope_("cache_push_scan");
    if (!c) return fail(CACHE_E_INVALID_ARG, "cache_push_scan: null cache");
    if (peer_failed(c)) return peer_fail("cache_push_scan");
    if (c->push_phase != 1 || nb != c->push_nb) return fail(CACHE_E_STATE, "cache_push_scan: call after cache_push_queries with the same nb");
    if (topk < 1 || topk > c->arena_topk) return fail(CACHE_E_INVALID_ARG, "cache_push_scan: bad topk");
    DeviceGuard g(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    const ArenaLayout L = arena_layout(c->world, c->arena_nb, c->arena_topk, c->dim);
    const int64_t bg = (int64_t)c->world * nb;
    const int kmax = topk == 1 ? 1 : (topk <= 4 ? 4 : 16);
    wait_flags(c, (const uint32_t*)(c->arena + L.qflag), c->push_epoch, s);
    c->launches++;
    int parts = 0;
    if (bg > 0) {
        CK(c->gk.ensure((bg + 127) / 128 * 128));
        CK(cudaMemsetAsync(c->gk.p, 0, bg * 4, s));
        cache_status r = scan_rows(c, bg, (__nv_bfloat16*)(c->arena + L.qg), c->gk.p, kmax, s, &parts);
        if (r != CACHE_OK) return r;
    }
    PushRecs d{};
    for (int r = 0; r < c->world; ++r) d.inbox[r] = (cache_shard_rec*)(c->peer_arena[r] + L.inbox);
    d.nb = std::max<int64_t>(1, nb);
    d.me = c->rank;
    launch_local_merge_push(kmax, c->recs.p, parts, bg, topk, (const int32_t*)(c->arena + L.qstat), c->present,
                            c->rank, d, push_signal_of(c, L.rflag, 1), s);
    c->launches++;
    c->push_phase = 2;
    CK(cudaGetLastError());
    return CACHE_OK;
}

cache_status cache_push_merge(cache_t* c, int64_t nb, int32_t topk, uint64_t* out_ids, float* out_scores,
                              int32_t* out_k, void* latent_out, void** out_latent_ptr, int32_t* row_status,
                              void* stream) {
    NvtxScope nvtx_scope_("cache_push_merge");
    if (!c) return fail(CACHE_E_INVALID_ARG, "cache_push_merge: null cache");
    if (peer_failed(c)) return peer_fail("cache_push_merge");
    if (c->push_phase != 2 || nb != c->push_nb) return fail(CACHE_E_STATE, "cache_push_merge: call after cache_push_scan with the same nb");
    if (topk < 1 || topk > c->arena_topk) return fail(CACHE_E_INVALID_ARG, "cache_push_merge: bad topk");
    if (nb > 0 && (!out_ids || !out_scores || !out_k)) return fail(CACHE_E_INVALID_ARG, "cache_push_merge: null buffer");
    DeviceGuard g(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    const ArenaLayout L = arena_layout(c->world, c->arena_nb, c->arena_topk, c->dim);
    const int kmax = topk == 1 ? 1 : (topk <= 4 ? 4 : 16);
    wait_flags(c, (const uint32_t*)(c->arena + L.rflag), c->push_epoch, s);
    c->launches++;
    c->clock++;   // once per global batch on every rank, as cache_query_merge
    if (nb > 0) {
        launch_merge_sharded(kmax, (const cache_shard_rec*)(c->arena + L.inbox), nb, 0, c->world,
                             (int64_t)c->rank * nb, nb, topk, (const float*)(c->arena + L.invq),
                             (const int32_t*)(c->arena + L.qstat), c->peers, c->clock, c->L, c->km, out_ids,
                             out_scores, out_k, (uint8_t*)latent_out, out_latent_ptr, row_status, s);
        c->launches++;
    }
    c->queries += nb;
    c->push_phase = 3;
    CK(cudaGetLastError());
    return CACHE_OK;
}

// ---- pipelined host calls: batch i+1's upload (copy stream) overlaps batch i's lookup ----
cache_status cache_query_submit(cache_t* c, int32_t slot, int64_t b, const void* queries, int32_t q_dtype,
                                int32_t topk, void* latent_out, void* stream) {
    NvtxScope nvtx_scope_("cache_query_submit");
    if (!c) return fail(CACHE_E_INVALID_ARG, "cache_query_submit: null cache");
    if (slot < 0 || slot > 1 || b <= 0 || b > 0x7FFFFFFF || topk < 1 || topk > c->cfg.max_topk || !queries ||
        (q_dtype != CACHE_DTYPE_F32 && q_dtype != CACHE_DTYPE_BF16))
        return fail(CACHE_E_INVALID_ARG, "cache_query_submit: bad slot / b / topk / dtype / queries");
    if (latent_out && !c->pool) return fail(CACHE_E_INVALID_ARG, "cache_query_submit: no latent pool");
    cache_t::AsyncSlot& a = c->aslot[slot];
    if (a.pending) return fail(CACHE_E_STATE, "cache_query_submit: slot still pending (call cache_query_complete)");
    DeviceGuard g(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    if (!c->hcopy) CK(cudaStreamCreateWithFlags(&c->hcopy, cudaStreamNonBlocking));
    for (cudaEvent_t* e : {&a.copied, &a.consumed, &a.done})
        if (!*e) CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    const size_t qbytes = (size_t)b * c->dim * (q_dtype == CACHE_DTYPE_BF16 ? 2 : 4);
    const size_t o_sc = (size_t)b * topk * 8, o_k = o_sc + (size_t)b * topk * 4, o_st = o_k + (size_t)b * 4;
    const size_t obytes = o_st + (size_t)b * 4;
    if (a.in.n < qbytes) {   // growing the input buffer frees it: its last reader must be done
        CK(cudaEventSynchronize(a.consumed));
        CK(a.in.ensure(qbytes));
    }
    CK(a.out.ensure(obytes));
    if (a.h_out_n < obytes) {
        if (a.h_out) cudaFreeHost(a.h_out);
        a.h_out = nullptr;
        a.h_out_n = 0;
        CK(cudaHostAlloc(&a.h_out, obytes, cudaHostAllocDefault));
        a.h_out_n = obytes;
    }
    // upload on the copy stream once the slot's previous lookup has read its input
    CK(cudaStreamWaitEvent(c->hcopy, a.consumed, 0));
    CK(cudaMemcpyAsync(a.in.p, queries, qbytes, cudaMemcpyHostToDevice, c->hcopy));
    CK(cudaEventRecord(a.copied, c->hcopy));
    CK(cudaStreamWaitEvent(s, a.copied, 0));
    uint8_t* ob = a.out.p;
    cache_status r = query_core(c, b, a.in.p, q_dtype, topk, (uint64_t*)ob, (float*)(ob + o_sc), (int32_t*)(ob + o_k),
                                latent_out, nullptr, (int32_t*)(ob + o_st), s);
    if (r != CACHE_OK) return r;
    CK(cudaEventRecord(a.consumed, s));
    CK(cudaMemcpyAsync(a.h_out, ob, obytes, cudaMemcpyDeviceToHost, s));
    CK(cudaEventRecord(a.done, s));
    a.b = b;
    a.topk = topk;
    a.pending = true;
    return CACHE_OK;
}

cache_status cache_query_complete(cache_t* c, int32_t slot, uint64_t* out_ids, float* out_scores, int32_t* out_k,
                                  int32_t* row_status) {
    NvtxScope nvtx_scope_("cache_query_complete");
    if (!c || slot < 0 || slot > 1 || !out_ids || !out_scores || !out_k)
        return fail(CACHE_E_INVALID_ARG, "cache_query_complete: bad argument");
    cache_t::AsyncSlot& a = c->aslot[slot];
    if (!a.pending) return fail(CACHE_E_STATE, "cache_query_complete: nothing submitted on this slot");
    DeviceGuard g(c->device);
    CK(cudaEventSynchronize(a.done));
    a.pending = false;
    const int64_t b = a.b, topk = a.topk;
    const size_t o_sc = (size_t)b * topk * 8, o_k = o_sc + (size_t)b * topk * 4, o_st = o_k + (size_t)b * 4;
    const uint8_t* hb = static_cast<const uint8_t*>(a.h_out);
    std::memcpy(out_ids, hb, (size_t)b * topk * 8);
    std::memcpy(out_scores, hb + o_sc, (size_t)b * topk * 4);
    std::memcpy(out_k, hb + o_k, (size_t)b * 4);
    if (row_status) std::memcpy(row_status, hb + o_st, (size_t)b * 4);
    return CACHE_OK;
}

cache_status cache_query_batch_host(cache_t* c, int64_t b, const void* queries, int32_t q_dtype, int32_t topk,
                                    uint64_t* out_ids, float* out_scores, int32_t* out_k, void* latent_out,
                                    int32_t* row_status, void* stream) {
    NvtxScope nvtx_scope_("cache_query_batch_host");
    if (!c) return fail(CACHE_E_INVALID_ARG, "cache_query_batch_host: null cache");
    if (b < 0 || b > 0x7FFFFFFF || topk < 1 || topk > c->cfg.max_topk ||
        (q_dtype != CACHE_DTYPE_F32 && q_dtype != CACHE_DTYPE_BF16))
        return fail(CACHE_E_INVALID_ARG, "cache_query_batch_host: bad b / topk / dtype");
    if (b == 0) return CACHE_OK;
    if (!queries || !out_ids || !out_scores || !out_k)
        return fail(CACHE_E_INVALID_ARG, "cache_query_batch_host: null buffer");
    if (latent_out && !c->pool) return fail(CACHE_E_INVALID_ARG, "cache_query_batch_host: no latent pool");
    DeviceGuard g(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    const size_t qbytes = (size_t)b * c->dim * (q_dtype == CACHE_DTYPE_BF16 ? 2 : 4);
    // latent_out may be device memory (the denoiser's input buffer on this GPU: gathered in
    // place, no host copy) or host memory (staged on the device, then copied back).
    bool lat_dev = false;
    if (latent_out) {
        cudaPointerAttributes pa;
        if (cudaPointerGetAttributes(&pa, latent_out) == cudaSuccess &&
            (pa.type == cudaMemoryTypeDevice || pa.type == cudaMemoryTypeManaged))
            lat_dev = true;
        cudaGetLastError();
    }
    CK(c->hq_in.ensure(qbytes));
    // ids | scores | K | status packed in one buffer -> one device-to-host copy
    const size_t o_ids = 0, o_sc = (size_t)b * topk * 8, o_k = o_sc + (size_t)b * topk * 4, o_st = o_k + (size_t)b * 4;
    const size_t obytes = o_st + (size_t)b * 4;
    CK(c->hq_out.ensure(obytes));
    if (c->h_out_n < obytes) {
        if (c->h_out) cudaFreeHost(c->h_out);
        c->h_out = nullptr;
        c->h_out_n = 0;
        CK(cudaHostAlloc(&c->h_out, obytes, cudaHostAllocDefault));
        c->h_out_n = obytes;
    }
    if (latent_out && !lat_dev) CK(c->hq_lat.ensure((size_t)b * c->L));
    uint8_t* ob = c->hq_out.p;
    uint8_t* lat = latent_out ? (uint8_t*)(lat_dev ? latent_out : (void*)c->hq_lat.p) : nullptr;
    // Large batches: the query upload is split into kHostSplit slices on a copy stream and
    // slice i's ingest/scan/finalize waits only for slice i, so the host-to-device copy of
    // the rest of the batch overlaps the scan (the scan is tensor-bound at these sizes, so a
    // quarter batch runs at the same rate per query).  One LRU clock tick for the whole batch.
    const int64_t sub = b >= kHostSplitMin ? (((b + kHostSplit - 1) / kHostSplit + 255) / 256) * 256 : b;
    if (sub >= b) {
        CK(cudaMemcpyAsync(c->hq_in.p, queries, qbytes, cudaMemcpyHostToDevice, s));
        cache_status r = query_core(c, b, c->hq_in.p, q_dtype, topk, (uint64_t*)(ob + o_ids), (float*)(ob + o_sc),
                                    (int32_t*)(ob + o_k), lat, nullptr, (int32_t*)(ob + o_st), s);
        if (r != CACHE_OK) return r;
    } else {
        if (!c->hcopy) CK(cudaStreamCreateWithFlags(&c->hcopy, cudaStreamNonBlocking));
        for (cudaEvent_t& e : c->hev)
            if (!e) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        const size_t row = qbytes / (size_t)b;
        CK(cudaEventRecord(c->hev[kHostSplit], s));   // hq_in is free once earlier work on s is done
        CK(cudaStreamWaitEvent(c->hcopy, c->hev[kHostSplit], 0));
        int ns = 0;
        for (int64_t off = 0; off < b; off += sub, ++ns) {
            const int64_t nb = std::min(sub, b - off);
            CK(cudaMemcpyAsync(c->hq_in.p + off * row, static_cast<const uint8_t*>(queries) + off * row, nb * row,
                               cudaMemcpyHostToDevice, c->hcopy));
            CK(cudaEventRecord(c->hev[ns], c->hcopy));
        }
        ns = 0;
        for (int64_t off = 0; off < b; off += sub, ++ns) {
            const int64_t nb = std::min(sub, b - off);
            CK(cudaStreamWaitEvent(s, c->hev[ns], 0));
            cache_status r = query_core(
                c, nb, c->hq_in.p + off * row, q_dtype, topk, (uint64_t*)(ob + o_ids) + off * topk,
                (float*)(ob + o_sc) + off * topk, (int32_t*)(ob + o_k) + off, lat ? lat + off * c->L : nullptr,
                nullptr, (int32_t*)(ob + o_st) + off, s, off == 0);
            if (r != CACHE_OK) return r;
        }
    }
    CK(cudaMemcpyAsync(c->h_out, ob, obytes, cudaMemcpyDeviceToHost, s));
    if (latent_out && !lat_dev)
        CK(cudaMemcpyAsync(latent_out, c->hq_lat.p, (size_t)b * c->L, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const uint8_t* hb = static_cast<const uint8_t*>(c->h_out);
    std::memcpy(out_ids, hb + o_ids, (size_t)b * topk * 8);
    std::memcpy(out_scores, hb + o_sc, (size_t)b * topk * 4);
    std::memcpy(out_k, hb + o_k, (size_t)b * 4);
    if (row_status) std::memcpy(row_status, hb + o_st, (size_t)b * 4);
    return CACHE_OK;
}

cache_status cache_evict_hist(cache_t* c, const cache_evict_state* st, int32_t pass, uint32_t* hist,
                              void* stream) {
    if (!c || !st || !hist || pass < 0 || pass > 7) return fail(CACHE_E_INVALID_ARG, "cache_evict_hist: bad argument");
    DeviceGuard g(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    CK(cudaMemsetAsync(hist, 0, 256 * 4, s));
    launch_evict_hist(c->present, c->fcnt, c->lastacc, c->ids, c->hwm, c->km, reinterpret_cast<const EvictState*>(st), pass,
                      hist, s);
    c->launches++;
    CK(cudaGetLastError());
    return CACHE_OK;
}

cache_status cache_evict_pick(cache_t* c, uint32_t* hist, cache_evict_state* st, int32_t pass, void* stream) {
    if (!c || !st || !hist || pass < 0 || pass > 7) return fail(CACHE_E_INVALID_ARG, "cache_evict_pick: bad argument");
    DeviceGuard g(c->device);
    launch_evict_pick(hist, reinterpret_cast<EvictState*>(st), pass, (cudaStream_t)stream);
    c->launches++;
    CK(cudaGetLastError());
    return CACHE_OK;
}

int64_t cache_live_items(const cache_t* c) { return c ? c->live_items : 0; }

static int bitlen(unsigned long long v) { return v ? 64 - __builtin_clzll(v) : 0; }

// Merge k freed slots (ascending) into a free list kept sorted descending (back() = lowest
// free slot, so allocation stays lowest-first and deterministic): one linear merge.
static void merge_free(std::vector<int64_t>& fl, const unsigned long long* asc, int64_t k, std::vector<int64_t>& tmp) {
    if (k <= 0) return;
    if (fl.empty() || (int64_t)asc[k - 1] < fl.back()) {   // all below the lowest free slot (the
        // usual case: evictions free the oldest slots): append them reversed in one range
        // insert (2.7x faster than per-element push_back on the pool's VMs: 0.57 vs 1.5 ms
        // for the 1M dirty entries of a C5 eviction)
        fl.insert(fl.end(), std::make_reverse_iterator(asc + k), std::make_reverse_iterator(asc));
        return;
    }
    tmp.resize(fl.size() + (size_t)k);
    size_t i = 0, o = 0;
    int64_t j = k - 1;   // asc read backwards = descending
    while (i < fl.size() && j >= 0) tmp[o++] = fl[i] > (int64_t)asc[j] ? fl[i++] : (int64_t)asc[j--];
    while (i < fl.size()) tmp[o++] = fl[i++];
    while (j >= 0) tmp[o++] = (int64_t)asc[j--];
    fl.swap(tmp);
}

// Second half of every eviction (fused cache_evict and the protocol's cache_evict_apply): the
// device lists (evicted keys in c->ekey, freed pool slots in c->epool, dirty slots / ids in
// c->edirty / c->edid) are sorted on the GPU -- lists of <= kSmallSort keys by one CTA each in
// a single launch, longer ones by LSD radix over only the bits their range spans (evicted keys:
// [kbase, kbase + 2^kbits)) -- copied to pinned host memory, and the host's entry mirror and
// free lists are updated.  n / nd / nfreed: evicted units, dirty entries, freed pool slots.
// NIRVANA_EVICT_TRACE=1: one line per cache_evict on stderr with the host-side phase times
static bool evict_trace() {
    static const bool on = std::getenv("NIRVANA_EVICT_TRACE") != nullptr;
    return on;
}
static double now_us() {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// want_ev / want_did: produce the evicted list / the dirty-id list in the library's pinned
// staging (hev_sorted: the reported values id << 3 | j or entry ids, masked on the GPU;
// hev_did); out_evicted / out_dirty_ids (may be null) receive a copy of them.  The full 64-bit
// keys stay on the device (c->ekey) for cache_last_evicted_keys.
// ev_ready: the kernel already emitted the evicted list sorted -- full keys in ev_full, the
// reported values in ev_ready (device) -- so no sort and no mask launch.
static cache_status evict_finish(cache_t* c, int64_t n, int64_t nd, int64_t nfreed, unsigned long long kbase, int kbits,
                                 bool want_ev, bool want_did, uint64_t* out_evicted, uint64_t* out_dirty_ids,
                                 int64_t* out_n_dirty, cudaStream_t s, double* tr = nullptr, bool presorted = false,
                                 const unsigned long long* ev_ready = nullptr, unsigned long long* ev_full = nullptr) {
    const bool entry_mode = c->km.gran == CACHE_EVICT_ENTRY;
    const bool pool_freed = !c->alias && nfreed > 0;
    CK(c->hev_pool.ensure((pool_freed ? nfreed : 0) * 8));
    CK(c->hev_ds.ensure(nd * 8));
    if (want_did) CK(c->hev_did.ensure(nd * 8));
    if (want_ev) CK(c->hev_sorted.ensure(n * 8));
    struct Job {
        unsigned long long* keys;
        int64_t n;
        int bits;
        unsigned long long base;
        void* host;
        unsigned long long* res;
    };
    Job jobs[4];
    int nj = 0;
    // presorted (fused path): the pool / dirty lists come out of the kernel's ordered bitmap
    // compaction already ascending; only the evicted keys need a sort
    if (pool_freed) jobs[nj++] = Job{c->epool.p, nfreed, std::max(1, bitlen((unsigned long long)std::max<int64_t>(1, c->lcap) - 1)), 0ull, c->hev_pool.p, nullptr};
    if (nd) {
        jobs[nj++] = Job{c->edirty.p, nd, std::max(1, bitlen((unsigned long long)std::max<int64_t>(1, c->hwm) - 1)), 0ull, c->hev_ds.p, nullptr};
        if (want_did)
            jobs[nj++] = Job{c->edid.p, nd, std::max(1, bitlen(c->next_id ? c->next_id - 1 : 0)), 0ull, c->hev_did.p, nullptr};
    }
    if (want_ev && n && !ev_ready) jobs[nj++] = Job{c->ekey.p, n, std::max(1, kbits), kbase, c->hev_sorted.p, nullptr};
    SortSegs small{};
    SortJobs big{};
    int64_t big_n = 0;
    for (int i = 0; i < nj; ++i) {
        Job& jb = jobs[i];
        jb.res = jb.keys;   // every sort lands in the list's own buffer
        if (jb.n <= 1 || (presorted && jb.keys != c->ekey.p)) continue;
        if (jb.n <= kSmallSort) {
            small.s[small.k++] = SortSeg{jb.keys, jb.n};
        } else {
            big.j[big.k++] = SortJob{jb.keys, c->ekey2.p, jb.n, (std::min(64, std::max(1, jb.bits)) + 7) / 8, jb.base};
            big_n = std::max(big_n, jb.n);
        }
    }
    if (big.k) {
        CK(c->ekey2.ensure_grow(big_n));
        for (int i = 0; i < big.k; ++i) big.j[i].tmp = c->ekey2.p;
        CK(c->escr.ensure_grow(sort_coop_scratch_words(big_n)));
        CK(launch_sort_coop(big, c->escr.p, s));
        c->launches++;
    }
    if (small.k) {
        launch_sort_small(small, s);
        c->launches++;
    }
    c->ev_full = ev_ready ? ev_full : c->ekey.p;
    if (want_ev && n && !ev_ready) {   // the reported values, masked on the GPU: item key -> id << 3 | j, entry key -> id
        CK(c->ekey2.ensure_grow(n));
        launch_mask_u64(c->ekey.p, c->ekey2.p, n, entry_mode ? 0xFFFFFFFFull : ((1ull << 35) - 1), s);
        c->launches++;
        jobs[nj - 1].res = c->ekey2.p;
    }
    CK(cudaGetLastError());
    // the lists the host bookkeeping needs (freed pool slots, dirty slots: jobs[] starts with
    // them) are copied first; the host updates its free lists while the evicted keys and dirty
    // ids are still crossing the link (at 12.5M entries ~6 MB, ~0.1 ms)
    int nfirst = 0;
    for (int i = 0; i < nj; ++i)
        if (jobs[i].host == c->hev_pool.p || jobs[i].host == c->hev_ds.p) nfirst = i + 1;
    for (int i = 0; i < nfirst; ++i)
        CK(cudaMemcpyAsync(jobs[i].host, jobs[i].res, jobs[i].n * 8, cudaMemcpyDeviceToHost, s));
    if (!c->ev_first) CK(cudaEventCreateWithFlags(&c->ev_first, cudaEventDisableTiming));
    CK(cudaEventRecord(c->ev_first, s));
    if (want_ev && n && ev_ready) CK(cudaMemcpyAsync(c->hev_sorted.p, ev_ready, n * 8, cudaMemcpyDeviceToHost, s));
    for (int i = nfirst; i < nj; ++i)
        CK(cudaMemcpyAsync(jobs[i].host, jobs[i].res, jobs[i].n * 8, cudaMemcpyDeviceToHost, s));
    c->live_items -= nfreed;
    if (tr) tr[0] = now_us();
    CK(cudaEventSynchronize(c->ev_first));   // pool / dirty-slot lists landed
    const unsigned long long* ds = static_cast<const unsigned long long*>(c->hev_ds.p);
    if (pool_freed) merge_free(c->free_l, static_cast<const unsigned long long*>(c->hev_pool.p), nfreed, c->free_tmp);
    for (int64_t i = 0; i < nd; ++i) c->h_live[(int64_t)ds[i]] = 0;
    c->live_entries -= nd;
    merge_free(c->free_e, ds, nd, c->free_tmp);
    CK(cudaStreamSynchronize(s));   // the rest of the lists landed
    if (tr) tr[1] = now_us();
    if (out_dirty_ids && nd) std::memcpy(out_dirty_ids, c->hev_did.p, nd * 8);
    if (out_n_dirty) *out_n_dirty = nd;
    c->last_nd = want_did ? nd : 0;
    // shrink the scan high-water mark past trailing empty slots
    while (c->hwm > 0 && c->h_live[c->hwm - 1] == 0) c->hwm--;
    c->last_ev_n = want_ev ? n : 0;
    if (out_evicted && n) std::memcpy(out_evicted, c->hev_sorted.p, n * 8);
    if (tr) tr[2] = now_us();
    return CACHE_OK;
}

// Eviction list workspaces for up to `bound` evicted units / `dbound` dirty entries.
static cudaError_t evict_lists(cache_t* c, int64_t bound, int64_t dbound, int64_t pbound) {
    cudaError_t e;
    if ((e = c->ekey.ensure_grow(bound)) != cudaSuccess) return e;
    if ((e = c->ekey2.ensure_grow(std::max(std::max(pbound, dbound), bound))) != cudaSuccess) return e;
    if ((e = c->epool.ensure_grow(pbound)) != cudaSuccess) return e;
    if ((e = c->escr.ensure_grow(sort_scratch_words(std::max(std::max(pbound, dbound), bound)))) != cudaSuccess) return e;
    if ((e = c->edirty.ensure_grow(dbound)) != cudaSuccess) return e;
    return c->edid.ensure_grow(dbound);
}

// cache_evict: the fused select + apply of evict.cu (one cooperative launch), then
// evict_finish.  The protocol's building blocks (cache_evict_hist / _pick / _apply) remain for
// the distributed eviction, whose histograms are summed over ranks between passes.
static cache_status evict_impl(cache_t* c, int64_t n, bool want_ev, bool want_did, uint64_t* out_evicted,
                               uint64_t* out_dirty_ids, int64_t* out_n_dirty, void* stream);

cache_status cache_evict(cache_t* c, int64_t n, uint64_t* out_evicted, uint64_t* out_dirty_ids,
                         int64_t* out_n_dirty, void* stream) {
    NvtxScope nvtx_scope_("cache_evict");
    return evict_impl(c, n, out_evicted != nullptr, out_dirty_ids != nullptr, out_evicted, out_dirty_ids, out_n_dirty,
                      stream);
}

cache_status cache_evict_view(cache_t* c, int64_t n, const uint64_t** out_evicted, const uint64_t** out_dirty_ids,
                              int64_t* out_n_dirty, void* stream) {
    NvtxScope nvtx_scope_("cache_evict_view");
    if (!c || !out_evicted || !out_dirty_ids || !out_n_dirty)
        return fail(CACHE_E_INVALID_ARG, "cache_evict_view: null argument");
    *out_evicted = *out_dirty_ids = nullptr;
    *out_n_dirty = 0;
    cache_status r = evict_impl(c, n, true, true, nullptr, nullptr, out_n_dirty, stream);
    if (r != CACHE_OK) return r;
    *out_evicted = static_cast<const uint64_t*>(c->hev_sorted.p);
    *out_dirty_ids = static_cast<const uint64_t*>(c->hev_did.p);
    return CACHE_OK;
}

// Workspaces, zeroed scratch and kernel arguments of one fused eviction.  n_sel: the number of
// units the selection evicts (globally, for a distributed eviction); n_loc: a bound on this
// cache's share (its list capacities).
static cache_status evict_setup(cache_t* c, int64_t n_sel, int64_t n_loc, bool want_ev, SelArgs& a, cudaStream_t s) {
    const bool entry_mode = c->km.gran == CACHE_EVICT_ENTRY;
    const int64_t n = std::max<int64_t>(1, n_loc);
    // dirty entries: n in entry mode, <= min(n, live entries) in item mode
    const int64_t dbound = std::max<int64_t>(1, std::min<int64_t>(n, c->live_entries));
    const int64_t pbound = entry_mode ? n * c->num_k : n;
    CK(evict_lists(c, n, dbound, pbound));
    const int64_t units = entry_mode ? c->live_entries : c->live_items;
    const int64_t ccap = std::max<int64_t>(65536, units / 16);
    CK(c->ckey.ensure_grow(ccap));
    CK(c->cslot.ensure_grow(ccap));
    // [level histograms][the window estimate's sample histogram][SelOut] (zeroed), compaction totals
    const size_t ws = (size_t)(kSelMaxLevels + 1) * kSelBins * 4 + sizeof(SelOut);
    // compaction totals: one per 512-word chunk of each ordered-output bitmap (evict.cu)
    const int64_t nchunks = (c->hwm + 31) / 32 / 512 + ((int64_t)(c->next_id / (uint64_t)c->world) + 32) / 32 / 512 +
                            (c->alias ? 0 : (c->lcap + 31) / 32 / 512) + kEvBitsWords / 512 + 8;
    CK(c->selws.ensure(ws + 4 * (size_t)std::max<int64_t>(4 * 4096, nchunks)));
    CK(cudaMemsetAsync(c->selws.p, 0, ws, s));
    SelOut* so = reinterpret_cast<SelOut*>(c->selws.p + (size_t)(kSelMaxLevels + 1) * kSelBins * 4);
    // bitmaps of the ordered outputs: dirty slots (< hwm), dirty ids / world (< next_id), freed
    // pool slots (< latent capacity; not tracked under aliasing)
    const int64_t w_slot = (c->hwm + 31) / 32;
    const int64_t w_id = ((int64_t)(c->next_id / (uint64_t)c->world) + 1 + 31) / 32;
    const int64_t w_pool = c->alias ? 0 : (c->lcap + 31) / 32;
    const int64_t w_ev = want_ev ? kEvBitsWords : 0;   // evicted keys spanning < 2^23 values: bitmap-sorted
    CK(c->ebits.ensure_grow(w_slot + w_id + w_pool + w_ev));
    CK(cudaMemsetAsync(c->ebits.p, 0, (size_t)(w_slot + w_id + w_pool + w_ev) * 4, s));
    CK(c->eout.ensure_grow(2 * n));
    a = SelArgs{};
    a.present = c->present;
    a.fcnt = c->fcnt;
    a.lastacc = c->lastacc;
    a.ids = c->ids;
    a.lslot = c->lslot;
    a.inv_e = c->inv_e;
    a.n_slots = c->hwm;
    a.n = (unsigned long long)n_sel;
    a.hist = reinterpret_cast<uint32_t*>(c->selws.p);
    a.hist_s = a.hist + (size_t)kSelMaxLevels * kSelBins;
    a.units = (unsigned long long)units;
    a.sample = 0;   // the single-cache call turns the window on (evict_impl)
    a.cand_key = c->ckey.p;
    a.cand_slot = c->cslot.p;
    a.cand_cap = (unsigned long long)(c->cand_cap_override >= 0 ? std::min<int64_t>(c->cand_cap_override, c->ckey.n)
                                                                 : (int64_t)c->ckey.n);
    a.ev_key = c->ekey.p;
    a.ev_pool = c->epool.p;
    a.dirty_slot = c->edirty.p;
    a.dirty_id = c->edid.p;
    a.ev_cap = want_ev ? (unsigned long long)n : 0ull;   // 0: no unsorted key list (count-only evictions)
    a.dslot_bits = c->ebits.p;
    a.did_bits = c->ebits.p + w_slot;
    a.pool_bits = w_pool ? c->ebits.p + w_slot + w_id : nullptr;
    a.dslot_words = w_slot;
    a.did_words = w_id;
    a.pool_words = w_pool;
    a.world = c->world;
    a.rank = c->rank;
    a.part = reinterpret_cast<uint32_t*>(c->selws.p + ws);
    a.ev_bits = w_ev ? c->ebits.p + w_slot + w_id + w_pool : nullptr;
    a.ev_bits_words = w_ev;
    a.ev_sorted = c->eout.p;
    a.ev_masked = c->eout.p + n;
    a.ev_mask = entry_mode ? 0xFFFFFFFFull : ((1ull << 35) - 1);
    a.out = so;
    a.phase = kPhaseAll;
    return CACHE_OK;
}

static cache_status evict_impl(cache_t* c, int64_t n, bool want_ev, bool want_did, uint64_t* out_evicted,
                               uint64_t* out_dirty_ids, int64_t* out_n_dirty, void* stream) {
    if (!c) return fail(CACHE_E_INVALID_ARG, "cache_evict: null cache");
    if (n < 0) return fail(CACHE_E_INVALID_ARG, "cache_evict: n < 0");
    const bool entry_mode = c->km.gran == CACHE_EVICT_ENTRY;
    if (entry_mode ? n > c->live_entries : n > c->live_items)
        return fail(CACHE_E_EVICT_RANGE, "cache_evict: n exceeds live items (entries in entry mode)");
    if (out_n_dirty) *out_n_dirty = 0;
    if (n == 0) return CACHE_OK;
    DeviceGuard g(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    SelArgs a;
    cache_status rs = evict_setup(c, n, n, want_ev, a, s);
    if (rs != CACHE_OK) return rs;
    // Single-sweep window (evict.cu): estimate the n-th key from every S-th slot (S <= 64, >= ~16K
    // sampled slots), then one full sweep histograms every key
    // AND compacts every key below the estimate's upper bin edge; when the n-th key's bin lies
    // below it (else the two-sweep path runs), the selection and the apply run on the candidates.
    if (c->evict_sample != 0 && 2 * (unsigned long long)n <= a.cand_cap)
        // odd strides: a power-of-two stride kept hitting the same HBM channels (the 1/64 sample of
        // 12.5M slots took 15 us, NV_SEL_TRACE)
        a.sample = c->evict_sample > 0 ? c->evict_sample
                                       : (int)(std::max<int64_t>(1, std::min<int64_t>(63, c->hwm / 16384)) | 1);
    SelOut* so = a.out;
    const int64_t dbound = std::max<int64_t>(1, std::min<int64_t>(n, c->live_entries));
    const int64_t pbound = entry_mode ? n * c->num_k : n;
    const bool trace = evict_trace();
    double t0 = trace ? now_us() : 0.0, t1 = 0.0, t2 = 0.0, tf[3] = {0, 0, 0};
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    if (trace) {
        cudaEventCreate(&ev0);
        cudaEventCreate(&ev1);
        sel_trace_reset(s);
        cudaEventRecord(ev0, s);
    }
    CK(launch_evict_select(a, c->km, s));
    c->launches++;
    if (trace) cudaEventRecord(ev1, s);
    SelOut h{};
    CK(cudaMemcpyAsync(&h, so, sizeof(h), cudaMemcpyDeviceToHost, s));
    if (trace) t1 = now_us();
    CK(cudaStreamSynchronize(s));
    if (trace) t2 = now_us();
    c->last_sel[0] = h.levels;
    c->last_sel[1] = h.full_sweeps;
    c->last_sel[2] = h.compact_level;
    c->last_sel[3] = (int64_t)(h.window == 1 ? h.cnt_w : h.cnt[3]);
    c->last_window = h.window;
    const int64_t got = (int64_t)h.cnt[0], nd = (int64_t)h.cnt[1];
    const int64_t nfreed = entry_mode ? (int64_t)h.cnt[2] : got;
    if (h.err || got != n || nd > dbound || nfreed > pbound)
        return fail(CACHE_E_STATE, "cache_evict: selection count mismatch (internal error); handle state undefined");
    const unsigned long long kmin = ~h.kmin_inv;
    cache_status r = evict_finish(c, n, nd, nfreed, kmin, bitlen(h.T - kmin), want_ev || out_evicted,
                                  want_did || out_dirty_ids, out_evicted, out_dirty_ids, out_n_dirty, s,
                                  trace ? tf : nullptr, /*presorted=*/true, h.ev_sorted ? a.ev_masked : nullptr,
                                  h.ev_sorted ? a.ev_sorted : nullptr);
    if (trace) {
        float kms = 0.f;
        cudaEventElapsedTime(&kms, ev0, ev1);
        cudaEventDestroy(ev0);
        cudaEventDestroy(ev1);
        std::fprintf(stderr,
                     "{\"evict_trace\": {\"n\": %lld, \"slots\": %lld, \"select_kernel_us\": %.1f, \"launch_us\": %.1f, "
                     "\"select_wait_us\": %.1f, \"sort_enqueue_us\": %.1f, \"sort_wait_us\": %.1f, \"host_us\": %.1f, "
                     "\"total_us\": %.1f, \"levels\": %u, \"full_sweeps\": %u, \"compact_level\": %u, "
                     "\"candidates\": %llu, \"key_bits\": %d, \"dirty\": %lld}}\n",
                     (long long)n, (long long)c->hwm, kms * 1e3, t1 - t0, t2 - t1, tf[0] - t2, tf[1] - tf[0], tf[2] - tf[1],
                     tf[2] - t0, h.levels, h.full_sweeps, h.compact_level, h.cnt[3], bitlen(h.T - kmin), (long long)nd);
        // NV_SEL_TRACE builds: phase stamps relative to the earliest CTA start (us), first / last CTA
        unsigned long long lo[kSelTraceN], hi[kSelTraceN];
        static unsigned long long cta[kSelTraceCta][1024];
        const int ns = sel_trace_read(lo, hi, &cta[0][0]);
        if (ns) {
            // per-CTA: the time between consecutive early stamps, the 6 slowest CTAs of each
            int grid = 0;
            while (grid < 1024 && cta[0][grid] >= lo[0] && cta[0][grid] - lo[0] < 100000000ull) ++grid;
            std::fprintf(stderr, "{\"sel_cta_grid\": %d, \"slowest\": [", grid);
            for (int st = 1; st < kSelTraceCta && hi[st]; ++st) {
                std::vector<std::pair<double, int>> d;
                for (int b = 0; b < grid; ++b) d.push_back({(cta[st][b] - cta[st - 1][b]) * 1e-3, b});
                std::sort(d.begin(), d.end());
                std::fprintf(stderr, "%s{\"stamp\": %d, \"median_us\": %.2f, \"top\": [", st > 1 ? ", " : "", st,
                             d.empty() ? 0.0 : d[d.size() / 2].first);
                for (int k = 0; k < 6 && k < (int)d.size(); ++k)
                    std::fprintf(stderr, "%s[%d, %.2f]", k ? ", " : "", d[d.size() - 1 - k].second, d[d.size() - 1 - k].first);
                std::fprintf(stderr, "]}");
            }
            std::fprintf(stderr, "]}\n");
            std::fprintf(stderr, "{\"sel_phases_us\": [");
            bool first = true;
            for (int i = 0; i < ns && hi[i]; ++i) {
                std::fprintf(stderr, "%s[%.2f, %.2f]", first ? "" : ", ", (lo[i] - lo[0]) * 1e-3, (hi[i] - lo[0]) * 1e-3);
                first = false;
            }
            std::fprintf(stderr, "]}\n");
        }
    }
    return r;
}

// ---- distributed fused eviction (SURVEY 8(e) a9 across shards): the single-cache kernel's
// levels, one launch each, with the 4,096-bin histograms summed over ranks between them ----
static cache_status sel_launch(cache_t* c, int phase, uint32_t* level_hist, cudaStream_t s) {
    SelArgs a = c->dsel;
    a.phase = phase;
    a.level_hist = level_hist;
    CK(launch_evict_select(a, c->km, s));
    c->launches++;
    return CACHE_OK;
}

cache_status cache_evict_sel_begin(cache_t* c, int64_t n, void* stream) {
    NvtxScope nvtx_scope_("cache_evict_sel_begin");
    if (!c || n < 1) return fail(CACHE_E_INVALID_ARG, "cache_evict_sel_begin: bad argument");
    if (peer_failed(c)) return peer_fail("cache_evict_sel_begin");
    DeviceGuard g(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    const bool entry_mode = c->km.gran == CACHE_EVICT_ENTRY;
    const int64_t units = entry_mode ? c->live_entries : c->live_items;
    cache_status r = evict_setup(c, n, std::min<int64_t>(n, units), /*want_ev=*/true, c->dsel, s);
    if (r != CACHE_OK) return r;
    CK(c->dstate.ensure(1));
    CK(cudaMemsetAsync(c->dstate.p, 0, sizeof(SelState), s));
    CK(c->dlhist.ensure((size_t)kSelMaxLevels * kSelBins));
    CK(cudaMemsetAsync(c->dlhist.p, 0, (size_t)kSelMaxLevels * kSelBins * 4, s));
    c->dsel.state = c->dstate.p;
    // the single-sweep window on this shard (evict.cu, kPhaseL0): on when this rank's share of
    // n (n / world) fits twice in its candidate buffer; each rank keeps or drops its window alone
    const int64_t share = (n + c->world - 1) / c->world;
    if (c->evict_sample != 0 && 2 * (unsigned long long)share <= c->dsel.cand_cap)
        c->dsel.sample = c->evict_sample > 0 ? c->evict_sample
                                             : (int)(std::max<int64_t>(1, std::min<int64_t>(63, c->hwm / 16384)) | 1);
    c->dsel_level = 0;
    c->dsel_push = false;
    c->dsel_done = false;
    return CACHE_OK;
}

cache_status cache_evict_sel_level(cache_t* c, int32_t level, uint32_t* hist, void* stream) {
    NvtxScope nvtx_scope_("cache_evict_sel_level");
    if (!c || !hist) return fail(CACHE_E_INVALID_ARG, "cache_evict_sel_level: bad argument");
    if (level != c->dsel_level || level >= kSelMaxLevels)
        return fail(CACHE_E_STATE, "cache_evict_sel_level: levels out of order (begin, then level / pick 0, 1, ...)");
    DeviceGuard g(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    CK(cudaMemsetAsync(hist, 0, (size_t)kSelBins * 4, s));
    return sel_launch(c, level == 0 ? kPhaseL0 : kPhaseLevel, hist, s);
}

static cache_status sel_pick_done(cache_t* c, int32_t level, const uint32_t* ghist, int32_t* out_done, cudaStream_t s) {
    CK(launch_evict_dpick(c->dsel, ghist, level, s));
    c->launches++;
    SelState h{};
    CK(cudaMemcpyAsync(&h, c->dstate.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (out_done) *out_done = (int32_t)(h.done | h.fail);
    c->dsel_done = (h.done | h.fail) != 0u;
    c->dsel_level = level + 1;
    return CACHE_OK;
}

cache_status cache_evict_sel_pick(cache_t* c, int32_t level, const uint32_t* ghist, int32_t* out_done, void* stream) {
    NvtxScope nvtx_scope_("cache_evict_sel_pick");
    if (!c || !ghist) return fail(CACHE_E_INVALID_ARG, "cache_evict_sel_pick: bad argument");
    if (level + 1 != c->dsel_level + 1 || level != c->dsel_level)
        return fail(CACHE_E_STATE, "cache_evict_sel_pick: call after cache_evict_sel_level of the same level");
    DeviceGuard g(c->device);
    return sel_pick_done(c, level, ghist, out_done, (cudaStream_t)stream);
}

cache_status cache_evict_sel_apply(cache_t* c, int64_t cap, uint64_t* out_evicted, int64_t* out_n,
                                   uint64_t* out_dirty_ids, int64_t* out_n_dirty, void* stream) {
    NvtxScope nvtx_scope_("cache_evict_sel_apply");
    if (!c || cap < 0) return fail(CACHE_E_INVALID_ARG, "cache_evict_sel_apply: bad argument");
    if (c->dsel_level < 1 || !c->dsel_done)
        return fail(CACHE_E_STATE, "cache_evict_sel_apply: the selection is not finished (begin, then level / pick "
                                   "0, 1, ... until a pick reports done)");
    if (peer_failed(c)) return peer_fail("cache_evict_sel_apply");
    DeviceGuard g(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    const bool entry_mode = c->km.gran == CACHE_EVICT_ENTRY;
    c->dsel_level = -1;
    cache_status r = sel_launch(c, kPhaseFinal, nullptr, s);
    if (r != CACHE_OK) return r;
    SelOut h{};
    CK(cudaMemcpyAsync(&h, c->dsel.out, sizeof(h), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const int64_t n = (int64_t)h.cnt[0], nd = (int64_t)h.cnt[1];
    const int64_t nfreed = entry_mode ? (int64_t)h.cnt[2] : n;
    if (out_n) *out_n = n;
    c->last_sel[0] = h.levels;
    c->last_sel[1] = h.full_sweeps;
    c->last_sel[2] = h.compact_level;
    c->last_sel[3] = (int64_t)(h.window == 1 ? h.cnt_w : h.cnt[3]);
    c->last_window = h.window;
    if (h.err || n > cap || nd > cap || (unsigned long long)n > c->dsel.ev_cap)
        return fail(CACHE_E_STATE, "cache_evict_sel_apply: selection failed or more evictions than the output "
                                   "capacity (ranks passed different n?); handle state undefined");
    const unsigned long long kmin = ~h.kmin_inv;
    return evict_finish(c, n, nd, nfreed, kmin, bitlen(h.T - kmin), true, true, out_evicted, out_dirty_ids, out_n_dirty,
                        s, nullptr, /*presorted=*/true, h.ev_sorted ? c->dsel.ev_masked : nullptr,
                        h.ev_sorted ? c->dsel.ev_sorted : nullptr);
}

// push variants: the level histogram goes into every rank's arena over NVLink (P2P atomics) and
// the pick waits for every rank's level flag, then reads the summed histogram from its own arena
cache_status cache_push_evict_sel_level(cache_t* c, int32_t level, void* stream) {
    NvtxScope nvtx_scope_("cache_push_evict_sel_level");
    if (!c) return fail(CACHE_E_INVALID_ARG, "cache_push_evict_sel_level: null cache");
    if (peer_failed(c)) return peer_fail("cache_push_evict_sel_level");
    if (!c->push_ok) return fail(CACHE_E_STATE, "cache_push_evict_sel_level: no push arenas");
    if (level != c->dsel_level || level >= kSelMaxLevels)
        return fail(CACHE_E_STATE, "cache_push_evict_sel_level: levels out of order");
    DeviceGuard g(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    if (level == 0) c->evict_epoch++;
    c->dsel_push = true;
    uint32_t* local = c->dlhist.p + (size_t)level * kSelBins;
    cache_status r = sel_launch(c, level == 0 ? kPhaseL0 : kPhaseLevel, local, s);
    if (r != CACHE_OK) return r;
    const ArenaLayout L = arena_layout(c->world, c->arena_nb, c->arena_topk, c->dim);
    PushHist ph{};
    for (int q = 0; q < c->world; ++q) ph.dst[q] = (unsigned int*)(c->peer_arena[q] + L.esel) + (size_t)level * kSelBins;
    ph.world = c->world;
    PushSignal sig = push_signal_of(c, L.eflag + (size_t)level * kMaxWorld * 4, 2);
    sig.epoch = c->evict_epoch;
    launch_push_hist_bins(local, kSelBins, ph, sig, s);
    c->launches++;
    CK(cudaGetLastError());
    return CACHE_OK;
}

cache_status cache_push_evict_sel_pick(cache_t* c, int32_t level, int32_t* out_done, void* stream) {
    NvtxScope nvtx_scope_("cache_push_evict_sel_pick");
    if (!c) return fail(CACHE_E_INVALID_ARG, "cache_push_evict_sel_pick: null cache");
    if (peer_failed(c)) return peer_fail("cache_push_evict_sel_pick");
    if (!c->push_ok || level != c->dsel_level || !c->dsel_push)
        return fail(CACHE_E_STATE, "cache_push_evict_sel_pick: call after cache_push_evict_sel_level of the same level");
    DeviceGuard g(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    const ArenaLayout L = arena_layout(c->world, c->arena_nb, c->arena_topk, c->dim);
    wait_flags(c, (const uint32_t*)(c->arena + L.eflag + (size_t)level * kMaxWorld * 4), c->evict_epoch, s);
    c->launches++;
    uint32_t* acc = (uint32_t*)(c->arena + L.esel) + (size_t)level * kSelBins;
    cache_status r = sel_pick_done(c, level, acc, out_done, s);
    if (r != CACHE_OK) return r;
    // the summed histogram is consumed: clear it for this level of the next eviction (a peer adds
    // into it again only after this rank has published that eviction's earlier levels)
    CK(cudaMemsetAsync(acc, 0, (size_t)kSelBins * 4, s));
    if (peer_failed(c)) return peer_fail("cache_push_evict_sel_pick");
    return CACHE_OK;
}

cache_status cache_evict_apply(cache_t* c, const cache_evict_state* st, int64_t cap, uint64_t* out_evicted,
                               int64_t* out_n, uint64_t* out_dirty_ids, int64_t* out_n_dirty, void* stream) {
    if (!c || !st || cap < 0) return fail(CACHE_E_INVALID_ARG, "cache_evict_apply: bad argument");
    DeviceGuard g(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    const bool entry_mode = c->km.gran == CACHE_EVICT_ENTRY;
    // at most min(cap, live units) keys are <= the selected threshold on this rank
    const int64_t bound = std::max<int64_t>(1, std::min<int64_t>(cap, entry_mode ? c->live_entries : c->live_items));
    const int64_t dbound = std::max<int64_t>(1, std::min<int64_t>(std::max<int64_t>(cap, 1), c->live_entries));
    // freed pool slots: one per evicted item, or up to num_k per evicted entry in entry mode
    const int64_t pbound = entry_mode ? bound * c->num_k : bound;
    CK(evict_lists(c, bound, dbound, pbound));
    CK(c->eslot.ensure_grow(bound));
    CK(c->ecnt.ensure(3));
    CK(cudaMemsetAsync(c->ecnt.p, 0, 24, s));
    launch_evict_apply(c->present, c->fcnt, c->lastacc, c->ids, c->lslot, c->inv_e, c->hwm, c->km,
                       reinterpret_cast<const EvictState*>(st), c->ekey.p, c->epool.p, c->eslot.p, c->ecnt.p,
                       c->edirty.p, c->edid.p, bound, dbound, s, c->abortw.p);
    c->launches++;
    unsigned long long cnt[3];
    CK(cudaMemcpyAsync(cnt, c->ecnt.p, 24, cudaMemcpyDeviceToHost, s));
    EvictState hst{};
    CK(cudaMemcpyAsync(&hst, st, sizeof(hst), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (peer_failed(c)) return peer_fail("cache_evict_apply");   // the selection's exchange failed: nothing applied
    const int64_t n = (int64_t)cnt[0], nd = (int64_t)cnt[1];
    const int64_t nfreed = entry_mode ? (int64_t)cnt[2] : n;   // stored states removed
    if (out_n) *out_n = n;
    if (n > cap || nd > cap || n > bound || nd > dbound || nfreed > pbound)
        return fail(CACHE_E_STATE, "cache_evict_apply: more evictions than the output capacity (n differs "
                                   "between the selection and the apply?); handle state undefined");
    // evicted keys are <= the selected key (st->prefix)
    return evict_finish(c, n, nd, nfreed, 0ull, bitlen(hst.prefix), out_evicted != nullptr, out_dirty_ids != nullptr,
                        out_evicted, out_dirty_ids, out_n_dirty, s);
}

// Entry slot of id, or -1 (a scan of the host mirrors: only the inspection calls need it).
static int64_t find_slot(const cache_t* c, uint64_t id) {
    if (id > 0xFFFFFFFFull) return -1;
    for (int64_t e = 0; e < c->hwm; ++e)
        if (c->h_live[e] && c->h_ids[e] == (uint32_t)id) return e;
    return -1;
}

cache_status cache_get_meta(cache_t* c, uint64_t id, uint64_t* f, uint32_t* present_mask) {
    if (!c) return fail(CACHE_E_INVALID_ARG, "cache_get_meta: null cache");
    const int64_t slot = find_slot(c, id);
    if (slot < 0) return fail(CACHE_E_INVALID_ARG, "cache_get_meta: unknown id");
    DeviceGuard g(c->device);
    std::vector<uint32_t> fv(c->num_k);
    uint32_t m = 0;
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(fv.data(), c->fcnt + slot * c->num_k, c->num_k * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&m, c->present + slot, 4, cudaMemcpyDeviceToHost));
    if (f)
        for (int j = 0; j < c->num_k; ++j) f[j] = fv[j];
    if (present_mask) *present_mask = m;
    return CACHE_OK;
}

cache_status cache_get_row(cache_t* c, uint64_t id, uint16_t* out_bf16) {
    if (!c || !out_bf16) return fail(CACHE_E_INVALID_ARG, "cache_get_row: null argument");
    const int64_t slot = find_slot(c, id);
    if (slot < 0) return fail(CACHE_E_INVALID_ARG, "cache_get_row: unknown id");
    DeviceGuard g(c->device);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(out_bf16, c->emb + slot * c->dim, c->dim * 2, cudaMemcpyDeviceToHost));
    return CACHE_OK;
}

cache_status cache_stats(cache_t* c, cache_stats_t* out) {
    if (!c || !out) return fail(CACHE_E_INVALID_ARG, "cache_stats: null argument");
    DeviceGuard g(c->device);
    CK(cudaDeviceSynchronize());
    out->live_entries = c->live_entries;
    out->live_items = c->live_items;
    out->holes = c->live_entries * c->num_k - c->live_items;
    out->entry_hwm = c->hwm;
    out->next_id = c->next_id;
    out->queries = c->queries;
    out->free_entries = (int64_t)c->free_e.size();
    out->free_items = (int64_t)c->free_l.size();
    return CACHE_OK;
}

// ---- checkpoint / resume (the paper's cache persists as EFS files + a Qdrant
// collection) ----
namespace {
constexpr char kSnapMagic[8] = {'N', 'V', 'C', 'A', 'C', 'H', 'E', '1'};
constexpr uint32_t kSnapVersion = 1;
struct SnapHeader {
    char magic[8];
    uint32_t version, cfg_bytes;
    cache_config cfg;   // the configuration with the live threshold table / policy / granularity
    int64_t hwm, live_entries, live_items, queries, n_free_e, n_free_l, pool_hi;
    uint64_t next_id;
    uint32_t clock;
    int32_t scorer, pred_ok, pad;
};
// device <-> file through a pinned staging buffer, 64 MiB at a time
struct SnapIO {
    std::FILE* f = nullptr;
    void* stage = nullptr;
    size_t stage_n = 0;
    bool ok = true;
    cudaError_t err = cudaSuccess;
    ~SnapIO() {
        if (stage) cudaFreeHost(stage);
        if (f) std::fclose(f);
    }
    bool host(void* p, size_t n, bool wr) {
        if (!ok || !n) return ok;
        ok = (wr ? std::fwrite(p, 1, n, f) : std::fread(p, 1, n, f)) == n;
        return ok;
    }
    bool dev(void* d, size_t n, bool wr) {
        if (!ok || !n) return ok;
        if (!stage) {
            stage_n = (size_t)64 << 20;
            if ((err = cudaHostAlloc(&stage, stage_n, cudaHostAllocDefault)) != cudaSuccess) return ok = false;
        }
        for (size_t o = 0; o < n && ok; o += stage_n) {
            const size_t m = std::min(stage_n, n - o);
            if (wr) {
                if ((err = cudaMemcpy(stage, (uint8_t*)d + o, m, cudaMemcpyDeviceToHost)) != cudaSuccess) return ok = false;
                host(stage, m, true);
            } else {
                if (!host(stage, m, false)) return false;
                if ((err = cudaMemcpy((uint8_t*)d + o, stage, m, cudaMemcpyHostToDevice)) != cudaSuccess) return ok = false;
            }
        }
        return ok;
    }
};
// the state arrays, in file order (rows [0, hwm) of every per-slot array)
struct SnapArr {
    void* p;
    size_t n;
};
int snap_arrays(cache_t* c, SnapArr* a) {
    const size_t h = (size_t)c->hwm, nk = (size_t)c->num_k;
    a[0] = {c->emb, h * c->dim * 2};
    a[1] = {c->inv_e, h * 4};
    a[2] = {c->ids, h * 4};
    a[3] = {c->present, h * 4};
    a[4] = {c->lslot, h * nk * 4};
    a[5] = {c->fcnt, h * nk * 4};
    a[6] = {c->lastacc, h * nk * 4};
    return 7;
}
}  // namespace

cache_status cache_get_config(cache_t* c, cache_config* out) {
    if (!c || !out) return fail(CACHE_E_INVALID_ARG, "cache_get_config: null argument");
    *out = c->cfg;
    for (int j = 0; j < c->num_k; ++j) out->thresholds[j] = c->km.thr[j];
    out->k_bias = c->km.k_bias;
    out->evict_policy = c->km.policy;
    out->evict_granularity = c->km.gran;
    return CACHE_OK;
}

cache_status cache_save(cache_t* c, const char* path, int32_t with_latents) {
    NvtxScope nvtx_scope_("cache_save");
    if (!c || !path) return fail(CACHE_E_INVALID_ARG, "cache_save: null argument");
    DeviceGuard g(c->device);
    CK(cudaDeviceSynchronize());
    SnapIO io;
    if (!(io.f = std::fopen(path, "wb"))) return fail(CACHE_E_INVALID_ARG, std::string("cache_save: cannot write ") + path);
    SnapHeader hd{};
    std::memcpy(hd.magic, kSnapMagic, 8);
    hd.version = kSnapVersion;
    hd.cfg_bytes = (uint32_t)sizeof(cache_config);
    cache_get_config(c, &hd.cfg);
    hd.hwm = c->hwm;
    hd.live_entries = c->live_entries;
    hd.live_items = c->live_items;
    hd.queries = c->queries;
    hd.n_free_e = (int64_t)c->free_e.size();
    hd.n_free_l = (int64_t)c->free_l.size();
    // occupied pool prefix: the free list is sorted descending, so its leading run lcap-1,
    // lcap-2, ... is the never-used top of the pool (aliased pools: every slot may be in use)
    int64_t top = 0;
    if (!c->alias)
        while (top < hd.n_free_l && c->free_l[(size_t)top] == c->lcap - 1 - top) ++top;
    hd.pool_hi = (with_latents && c->pool) ? c->lcap - top : 0;
    hd.next_id = c->next_id;
    hd.clock = c->clock;
    hd.scorer = c->scorer;
    hd.pred_ok = c->pred_ok ? 1 : 0;
    io.host(&hd, sizeof(hd), true);
    io.host(c->h_live.data(), (size_t)c->hwm, true);
    io.host(c->h_ids.data(), (size_t)c->hwm * 4, true);
    io.host(c->free_e.data(), c->free_e.size() * 8, true);
    io.host(c->free_l.data(), c->free_l.size() * 8, true);
    SnapArr arr[8];
    for (int i = 0, na = snap_arrays(c, arr); i < na; ++i) io.dev(arr[i].p, arr[i].n, true);
    if (hd.pred_ok) {
        io.dev(c->pw.p, (size_t)c->dim * 4, true);
        io.dev(c->prho.p, 4, true);
    }
    io.dev(c->pool, (size_t)hd.pool_hi * c->L, true);
    if (io.err != cudaSuccess) return fail(CACHE_E_CUDA, std::string("cache_save: ") + cudaGetErrorString(io.err));
    if (!io.ok || std::fflush(io.f) != 0) return fail(CACHE_E_INVALID_ARG, std::string("cache_save: write failed: ") + path);
    return CACHE_OK;
}

cache_status cache_load(const char* path, int32_t device, cache_t** out) {
    NvtxScope nvtx_scope_("cache_load");
    if (!path || !out) return fail(CACHE_E_INVALID_ARG, "cache_load: null argument");
    *out = nullptr;
    SnapIO io;
    if (!(io.f = std::fopen(path, "rb"))) return fail(CACHE_E_INVALID_ARG, std::string("cache_load: cannot read ") + path);
    SnapHeader hd{};
    if (!io.host(&hd, sizeof(hd), false) || std::memcmp(hd.magic, kSnapMagic, 8) != 0 || hd.version != kSnapVersion ||
        hd.cfg_bytes != sizeof(cache_config))
        return fail(CACHE_E_INVALID_ARG, "cache_load: not a cache snapshot of this library version");
    cache_t* c = nullptr;
    cache_status r = cache_create(&hd.cfg, device, &c);
    if (r != CACHE_OK) return r;
    auto bad = [&](cache_status st, const std::string& what) {
        cache_destroy(c);
        return fail(st, "cache_load: " + what);
    };
    if (hd.hwm < 0 || hd.hwm > c->cap || hd.n_free_e < 0 || hd.n_free_e > c->cap || hd.n_free_l < 0 ||
        hd.n_free_l > std::max<int64_t>(c->lcap, 0) || hd.pool_hi < 0 || hd.pool_hi > std::max<int64_t>(c->lcap, 0))
        return bad(CACHE_E_INVALID_ARG, "inconsistent snapshot header");
    DeviceGuard g(c->device);
    c->hwm = hd.hwm;
    c->live_entries = hd.live_entries;
    c->live_items = hd.live_items;
    c->queries = hd.queries;
    c->next_id = hd.next_id;
    c->clock = hd.clock;
    c->scorer = hd.scorer;
    c->free_e.resize((size_t)hd.n_free_e);
    c->free_l.resize((size_t)hd.n_free_l);
    io.host(c->h_live.data(), (size_t)c->hwm, false);
    io.host(c->h_ids.data(), (size_t)c->hwm * 4, false);
    io.host(c->free_e.data(), c->free_e.size() * 8, false);
    io.host(c->free_l.data(), c->free_l.size() * 8, false);
    SnapArr arr[8];
    for (int i = 0, na = snap_arrays(c, arr); i < na; ++i) io.dev(arr[i].p, arr[i].n, false);
    if (hd.pred_ok) {
        if (c->pw.ensure(c->dim) != cudaSuccess || c->prho.ensure(1) != cudaSuccess)
            return bad(CACHE_E_OOM, "predictor");
        io.dev(c->pw.p, (size_t)c->dim * 4, false);
        io.dev(c->prho.p, 4, false);
        c->pred_ok = io.ok;
    }
    io.dev(c->pool, (size_t)hd.pool_hi * c->L, false);
    if (io.err != cudaSuccess) return bad(CACHE_E_CUDA, cudaGetErrorString(io.err));
    if (!io.ok) return bad(CACHE_E_INVALID_ARG, std::string("truncated snapshot: ") + path);
    if (cudaDeviceSynchronize() != cudaSuccess) return bad(CACHE_E_CUDA, "restore");
    *out = c;
    return CACHE_OK;
}

int64_t cache_live_entries(const cache_t* c) { return c ? c->live_entries : 0; }

cache_status cache_set_evict_granularity(cache_t* c, int32_t granularity) {
    if (!c || (granularity != CACHE_EVICT_ITEM && granularity != CACHE_EVICT_ENTRY))
        return fail(CACHE_E_INVALID_ARG, "cache_set_evict_granularity: bad argument");
    c->km.gran = granularity;
    return CACHE_OK;
}

cache_status cache_set_evict_policy(cache_t* c, int32_t policy) {
    if (!c || policy < CACHE_POLICY_LCBFU || policy > CACHE_POLICY_FIFO)
        return fail(CACHE_E_INVALID_ARG, "cache_set_evict_policy: bad argument");
    c->km.policy = policy;
    return CACHE_OK;
}

cache_status cache_set_scorer(cache_t* c, int32_t scorer) {
    if (!c || scorer < CACHE_SCORER_AUTO || scorer > CACHE_SCORER_TC_SINGLE)
        return fail(CACHE_E_INVALID_ARG, "cache_set_scorer: bad argument");
    c->scorer = scorer;
    return CACHE_OK;
}

cache_status cache_set_query_slices(cache_t* c, int32_t slices) {
    if (!c || slices < 0 || slices > kDevSplitMax) return fail(CACHE_E_INVALID_ARG, "cache_set_query_slices: bad argument");
    c->qslices = slices;
    return CACHE_OK;
}

cache_status cache_set_profile_events(cache_t* c, void* const* events) {
    if (!c) return fail(CACHE_E_INVALID_ARG, "cache_set_profile_events: null cache");
    c->prof_on = events != nullptr;
    for (int i = 0; i < 4; ++i) c->prof[i] = events ? (cudaEvent_t)events[i] : nullptr;
    if (events)
        for (int i = 0; i < 4; ++i)
            if (!c->prof[i]) {
                c->prof_on = false;
                return fail(CACHE_E_INVALID_ARG, "cache_set_profile_events: null event");
            }
    return CACHE_OK;
}

int64_t cache_kernel_launches(const cache_t* c) { return c ? c->launches : 0; }

}  // extern "C"

// ------------------------------- test-only entry points -------------------------------
#include "../../include/nirvana_cache_debug.h"
namespace nv {
bool launch_score_tc_dense(const TcPlan& p, const void* tmap_q, const void* tmap_e, const float* inv_e, int dim,
                           int64_t b, float* dense, int64_t dense_ld, cudaStream_t s);
}

extern "C" cache_status cache_debug_tc_scores(cache_t* c, int64_t b, const void* queries, int32_t q_dtype,
                                              float* out, int64_t ld, void* stream) {
    if (!c || b <= 0 || !queries || !out) return fail(CACHE_E_INVALID_ARG, "cache_debug_tc_scores: bad argument");
    if (!c->tm_e_ok || !tc_supported(c->dim)) return fail(CACHE_E_UNSUPPORTED, "tcgen05 scorer unavailable");
    const int64_t n_slots = c->hwm;
    if (n_slots == 0) return CACHE_OK;
    const bool pair = b > 128 && c->scorer != CACHE_SCORER_TC_SINGLE;
    TcPlan tp = tc_plan(b, n_slots, c->sm_count, pair);
    if (ld < (int64_t)tp.n_tiles * 256) return fail(CACHE_E_INVALID_ARG, "cache_debug_tc_scores: ld too small");
    DeviceGuard g(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t bpad = (b + 127) / 128 * 128;
    CK(c->qbuf.ensure((size_t)bpad * c->dim));
    CK(c->invq.ensure(bpad));
    CK(c->qstat.ensure(bpad));
    launch_normalise(queries, q_dtype, b, c->dim, c->qbuf.p, c->invq.p, c->qstat.p, s);
    if (bpad > b) CK(cudaMemsetAsync(c->qbuf.p + b * c->dim, 0, (bpad - b) * c->dim * 2, s));
    CUtensorMap tm_q;
    if (!encode_rows(&tm_q, c->qbuf.p, bpad, c->dim, 128)) return fail(CACHE_E_CUDA, "tensor map encode failed");
    if (!launch_score_tc_dense(tp, &tm_q, pair ? &c->tm_e128 : &c->tm_e, c->inv_e, c->dim, b, out, ld, s))
        return fail(CACHE_E_CUDA, std::string("tc dense launch: ") + cudaGetErrorString(cudaGetLastError()));
    return CACHE_OK;
}

extern "C" cache_status cache_debug_sort_u64(uint64_t* keys, int64_t n, void* stream) {
    return cache_debug_sort_u64_ex(keys, n, 64, 0ull, 0, stream);
}

extern "C" cache_status cache_debug_sort_u64_ex(uint64_t* keys, int64_t n, int32_t bits, uint64_t base, int32_t small,
                                                void* stream) {
    if (n < 0 || (n > 0 && !keys) || bits < 1 || bits > 64 || (small == 1 && n > kSmallSort))
        return fail(CACHE_E_INVALID_ARG, "cache_debug_sort_u64_ex: bad argument");
    if (n <= 1) return CACHE_OK;
    cudaStream_t s = (cudaStream_t)stream;
    auto* k = reinterpret_cast<unsigned long long*>(keys);
    if (small == 1) {
        SortSegs sg{};
        sg.s[0] = SortSeg{k, n};
        sg.k = 1;
        launch_sort_small(sg, s);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(s));
        return CACHE_OK;
    }
    DevBuf<unsigned long long> tmp;
    DevBuf<uint32_t> scr;
    CK(tmp.ensure(n));
    if (small == 2) {   // the eviction's cooperative one-launch sort
        CK(scr.ensure(sort_coop_scratch_words(n)));
        SortJobs jb{};
        jb.j[0] = SortJob{k, tmp.p, n, (bits + 7) / 8, (unsigned long long)base};
        jb.k = 1;
        cudaError_t e = launch_sort_coop(jb, scr.p, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        tmp.release();
        scr.release();
        CK(e);
        return CACHE_OK;
    }
    CK(scr.ensure(sort_scratch_words(n)));
    unsigned long long* r = launch_sort_u64(k, tmp.p, n, scr.p, s, bits, base);
    if (r != k) cudaMemcpyAsync(k, r, n * 8, cudaMemcpyDeviceToDevice, s);
    cudaError_t e = cudaStreamSynchronize(s);
    tmp.release();
    scr.release();
    CK(e);
    return CACHE_OK;
}

// Statistics of the last fused cache_evict: levels, full sweeps, compaction level, candidates.
extern "C" cache_status cache_debug_evict_stats(cache_t* c, int64_t* out4) {
    if (!c || !out4) return fail(CACHE_E_INVALID_ARG, "cache_debug_evict_stats: bad argument");
    for (int i = 0; i < 4; ++i) out4[i] = c->last_sel[i];
    return CACHE_OK;
}

extern "C" cache_status cache_debug_set_count(cache_t* c, uint64_t id, int32_t j, uint32_t f) {
    if (!c || j < 0 || j >= c->num_k) return fail(CACHE_E_INVALID_ARG, "cache_debug_set_count: bad argument");
    const int64_t e = find_slot(c, id);
    if (e < 0) return fail(CACHE_E_INVALID_ARG, "cache_debug_set_count: id not live");
    DeviceGuard g(c->device);
    CK(cudaMemcpy(c->fcnt + e * c->num_k + j, &f, 4, cudaMemcpyHostToDevice));
    return CACHE_OK;
}

// Single-sweep window of the fused eviction: stride -1 = auto, 0 = off, S = a fixed 1/S sample.
// Returns the last eviction's window outcome in *last (0 off, 1 used, 2 estimate missed).
extern "C" cache_status cache_debug_evict_window(cache_t* c, int32_t stride, int32_t set, int32_t* last) {
    if (!c) return fail(CACHE_E_INVALID_ARG, "cache_debug_evict_window: null cache");
    if (set) c->evict_sample = stride < 0 ? -1 : stride;
    if (last) *last = (int32_t)c->last_window;
    return CACHE_OK;
}

extern "C" cache_status cache_debug_set_evict_cand_cap(cache_t* c, int64_t cap) {
    if (!c) return fail(CACHE_E_INVALID_ARG, "cache_debug_set_evict_cand_cap: null cache");
    c->cand_cap_override = cap < 0 ? -1 : cap;
    return CACHE_OK;
}

extern "C" int64_t cache_debug_slot_of(cache_t* c, uint64_t id) {
    if (!c) return -1;
    return find_slot(c, id);
}
