// kernels.h -- launcher declarations shared by the host engine (cache.cu) and the kernels.
#pragma once
#include <algorithm>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "common.cuh"

namespace nv {

struct InsertPlan {          // one accepted insert row
    int64_t src_row;         // row index in the caller's batch / staging buffer
    int64_t slot;            // entry slot
    uint32_t id;             // assigned entry id
    uint32_t mask;           // present-K bitmask
    int32_t lslot[CACHE_MAX_K];  // latent-pool slot per K (-1 = not stored)
};

struct CopyPlan {            // one latent payload copy
    int64_t src_item;        // (row * num_k + j) in the caller's latents buffer
    int64_t dst_slot;        // latent-pool slot
};

struct EvictState {          // radix-select state (device); layout = cache_evict_state
    unsigned long long prefix;
    unsigned long long mask;
    unsigned long long remaining;
};

// gk (optional): per-row u32 reset to 0 (the scorer's global k-th-best gate, see score_tc.cu)
void launch_normalise(const void* x, int dtype, int64_t n, int dim, __nv_bfloat16* y, float* inv,
                      int32_t* status, cudaStream_t s, uint32_t* gk = nullptr);

int stream_parts(int64_t n_slots, int64_t b);
void launch_score_stream(int kmax, const __nv_bfloat16* emb, const float* inv_e, const uint32_t* ids,
                         int64_t n_slots, int dim, const __nv_bfloat16* qbuf, int64_t b, Rec* ws,
                         int parts, cudaStream_t s);

// tcgen05 scorer (score_tc.cu).  Returns false if the configuration is not supported.
struct TcPlan {
    int m_tiles;        // ceil(B / 128)
    int n_tiles;        // ceil(n_slots / 256)
    int chunk_tiles;    // n-tiles per chunk (top-k segment)
    int n_chunks;
    int grid;           // persistent CTAs (clusters for the CTA-pair kernel)
    int parts;          // records per query = n_chunks
    bool pair;          // cta_group::2 kernel: m_tiles counts 256-query tile pairs
};
bool tc_supported(int dim);
TcPlan tc_plan(int64_t b, int64_t n_slots, int sm_count, bool pair);
bool launch_score_tc(int kmax, const TcPlan& plan, const void* tmap_q, const void* tmap_e,
                     const float* inv_e, const uint32_t* ids, int dim, int64_t b, Rec* ws,
                     uint32_t* gk, cudaStream_t s);

// lastacc / clock: the LRU last-access clock of every hit item is set to `clock`
void launch_finalize(int kmax, const Rec* ws, int parts, int64_t B, int topk, const float* inv_q,
                     const int32_t* qstatus, const uint32_t* ids, const uint32_t* present,
                     const int32_t* lslot, uint32_t* fcnt, uint32_t* lastacc, uint32_t clock,
                     const uint8_t* pool, int64_t latent_bytes,
                     const KMap& km, uint64_t* out_ids, float* out_scores, int32_t* out_k,
                     uint8_t* latent_out, void** out_ptr, int32_t* out_status, cudaStream_t s,
                     bool pdl = true);

void launch_insert_commit(const __nv_bfloat16* ystage, const float* invstage, const InsertPlan* plan,
                          int64_t n_valid, int dim, int num_k, __nv_bfloat16* emb, float* inv_e,
                          uint32_t* ids, uint32_t* present, int32_t* lslot, uint32_t* fcnt, uint32_t* lastacc,
                          uint32_t clock, cudaStream_t s);
void launch_copy_latents(const uint8_t* src, const CopyPlan* plan, int64_t n, int64_t latent_bytes,
                         uint8_t* pool, cudaStream_t s);

void launch_evict_hist(const uint32_t* present, const uint32_t* fcnt, const uint32_t* lastacc, const uint32_t* ids,
                       int64_t n_slots, const KMap& km, const EvictState* st, int pass, unsigned int* hist,
                       cudaStream_t s);
void launch_evict_pick(unsigned int* hist, EvictState* st, int pass, cudaStream_t s);
void launch_evict_apply(uint32_t* present, uint32_t* fcnt, const uint32_t* lastacc, const uint32_t* ids,
                        const int32_t* lslot, float* inv_e, int64_t n_slots, const KMap& km, const EvictState* st,
                        unsigned long long* ev_key, unsigned long long* ev_pool, int64_t* ev_eslot,
                        unsigned long long* counters, unsigned long long* dirty_slot, unsigned long long* dirty_id,
                        int64_t ev_cap, int64_t dirty_cap, cudaStream_t s, const uint32_t* abort = nullptr);
// Ascending sort of n 64-bit keys with base <= key < base + 2^bits (LSD radix over key - base,
// ceil(bits/8) stable 8-bit passes); tmp: n keys, scratch: >= sort_scratch_words(n) u32.
// Returns the buffer that holds the result (keys or tmp).
int64_t sort_scratch_words(int64_t n);
unsigned long long* launch_sort_u64(unsigned long long* keys, unsigned long long* tmp, int64_t n, uint32_t* scratch,
                                    cudaStream_t s, int bits = 64, unsigned long long base = 0ull);
int sort_launches(int64_t n, int bits);
void launch_mask_u64(const unsigned long long* in, unsigned long long* out, int64_t n, unsigned long long mask,
                     cudaStream_t s);
// Up to 4 lists of <= kSmallSort keys, each sorted in place by one CTA (one launch).
constexpr int kSmallSort = 16384;
struct SortSeg {
    unsigned long long* keys;
    int64_t n;
};
struct SortSegs {
    SortSeg s[4];
    int k;
};
void launch_sort_small(const SortSegs& segs, cudaStream_t s);
// Up to 4 long lists sorted in ONE cooperative launch (sequentially, grid barriers between the
// LSD steps); each list's result lands in its keys buffer (tmp may be shared by the lists).
struct SortJob {
    unsigned long long* keys;
    unsigned long long* tmp;
    int64_t n;
    int passes;                  // ceil(bits / 8)
    unsigned long long base;     // keys in [base, base + 2^(8 passes))
};
struct SortJobs {
    SortJob j[4];
    int k;
};
int64_t sort_coop_scratch_words(int64_t max_n);
cudaError_t launch_sort_coop(const SortJobs& jobs, uint32_t* scratch, cudaStream_t s);

// Fused single-cache eviction (evict.cu): the exact n smallest unit keys selected and applied
// in ONE cooperative launch (see evict.cu for the algorithm).  `out` is zeroed by the caller.
struct SelOut {
    unsigned long long cnt[4];    // evicted units, dirty entries, freed pool slots (entry mode), candidates
    unsigned long long kmin_inv;  // ~(smallest live key)
    unsigned long long T;         // threshold: every unit with key <= T was evicted
    uint32_t levels, full_sweeps, compact_level, err;
    uint32_t ev_sorted, ev_over;  // evicted keys emitted sorted (bitmap path) / one fell beyond the bitmap
    unsigned long long cnt_w;     // single-sweep window: keys compacted by the level-0 sweep
    uint32_t window, pad;         // 0 off, 1 the selection ran on the window, 2 the estimate missed
    unsigned long long gnext[16]; // full sweeps (<= 9) of the single-cache launch: claimed tail groups
    unsigned long long whi;       // distributed level 0: this rank's window edge (0: none)
};
constexpr int kSelBins = 4096, kSelMaxLevels = 8;
// Selection state between the host-driven phases of the DISTRIBUTED fused eviction (each rank
// sweeps its shard, the 4,096-bin histograms are summed over ranks between phases, every rank
// picks identically).  Device memory, one per cache.
struct SelState {
    unsigned long long lo, T, kb, ev_lim;   // the SelLevel of the current level
    int w, shift, compact, pad0;
    unsigned long long rem, pcnt;           // rank wanted inside [lo, lo + 2^w), keys in it (global)
    long long ncand;                        // this rank's compacted candidates
    uint32_t done, fail, compacted, level, full, compact_level, pad1, pad2;   // pad1: window (0 off, 1 held, 2 missed)
};
enum { kPhaseAll = 0, kPhaseL0 = 1, kPhaseLevel = 2, kPhaseFinal = 3 };
struct SelArgs {
    uint32_t* present;
    uint32_t* fcnt;
    const uint32_t* lastacc;
    const uint32_t* ids;
    const int32_t* lslot;
    float* inv_e;
    int64_t n_slots;
    unsigned long long n;              // units to evict (<= live units)
    uint32_t* hist;                    // [kSelMaxLevels][kSelBins], zeroed by the caller
    uint32_t* hist_s;                  // [kSelBins] zeroed: the window estimate's sample histogram
    unsigned long long units;          // live units (the sample's rank scale)
    int sample;                        // single cache: window sample stride S (0: two-sweep path)
    unsigned long long* cand_key;      // candidate compaction buffers
    uint32_t* cand_slot;
    unsigned long long cand_cap;
    unsigned long long* ev_key;        // evicted unit keys (unsorted), capacity ev_cap
    unsigned long long* ev_pool;       // freed pool slots, ascending (from pool_bits)
    unsigned long long* dirty_slot;    // dirty entries: slots ascending, ids ascending
    unsigned long long* dirty_id;
    unsigned long long ev_cap;
    uint32_t* dslot_bits;              // zeroed bitmaps: dirty slots, dirty ids / world, freed
    uint32_t* did_bits;                //   pool slots (null: pool slots not tracked, aliasing)
    uint32_t* pool_bits;
    int64_t dslot_words, did_words, pool_words;
    int world, rank;                   // ids of this cache: id % world == rank
    uint32_t* part;                    // [4][grid] CTA totals of the compaction
    // evicted keys are unique: when they span < 32 * ev_bits_words values above the min key,
    // they are sorted by an ordered bitmap compaction in the kernel (no sort launches)
    uint32_t* ev_bits;                 // zeroed, ev_bits_words words (null: never)
    int64_t ev_bits_words;
    unsigned long long* ev_sorted;     // full keys, ascending
    unsigned long long* ev_masked;     // the reported values (key & ev_mask), ascending
    unsigned long long ev_mask;
    SelOut* out;
    // distributed phases (phase != kPhaseAll): the state, and this phase's LOCAL histogram
    // (zeroed by the caller; summed over ranks before the pick)
    int phase;
    SelState* state;
    uint32_t* level_hist;
};
cudaError_t launch_evict_select(const SelArgs& a, const KMap& km, cudaStream_t s);
// experiments (NV_SEL_TRACE=1 builds): per phase-stamp index, the earliest / latest CTA time
constexpr int kSelTraceN = 32, kSelTraceCta = 6;
void sel_trace_reset(cudaStream_t s);
// -> stamps compiled in (0: none); cta (may be null): [kSelTraceCta][1024] per-CTA times of the first stamps
int sel_trace_read(unsigned long long* tmin, unsigned long long* tmax, unsigned long long* cta);
// The pick of one distributed level from the rank-summed histogram ghist (every rank runs it
// with the same ghist, so every rank reaches the same state).
cudaError_t launch_evict_dpick(const SelArgs& a, const uint32_t* ghist, int level, cudaStream_t s);

// Cache-selector profiling (Alg. 2): per profiling query i with a live nearest entry
// (rec[i].key != 0), s_i = clamp(t_i * inv_q[i]); for every K_j with quality[j*b + i] <= alpha,
// fail[j] = max(fail[j], orderable(s_i)); smin = min over all valid i of orderable(s_i).
void launch_profile_reduce(const cache_shard_rec* recs, const float* inv_q, const int32_t* qstatus, int64_t b,
                           const float* quality, int num_k, float alpha, uint32_t* fail, uint32_t* smin,
                           cudaStream_t s);

// match predictor (predictor.cu)
void pred_margins(const __nv_bfloat16* emb, const float* inv_e, int64_t n_slots, int dim, const float* w,
                  uint32_t* keys, cudaStream_t s);
void pred_select(const uint32_t* keys, int64_t n, EvictState* st, unsigned int* hist, cudaStream_t s);
void pred_viol(const __nv_bfloat16* emb, const float* inv_e, const uint32_t* keys, int64_t n_slots, int dim,
               const EvictState* st, int all_rows, float* gpart, unsigned int* cpart, int nblk, cudaStream_t s);
void pred_update(const float* gpart, const unsigned int* cpart, int nblk, int dim, float* w, double nu, double eta,
                 int64_t n, int mode, cudaStream_t s);
void pred_finish(const EvictState* st, float* rho, cudaStream_t s);
void pred_predict(const __nv_bfloat16* qbuf, const float* inv_q, const int32_t* qstatus, int64_t b, int dim,
                  const float* w, const float* rho, uint8_t* flags, float* margin, cudaStream_t s);

// sharded lookup
constexpr int kMaxWorld = 16;
struct PeerPtrs {                       // per-rank device pointers (own rank included)
    const int32_t* lslot[kMaxWorld];
    uint32_t* fcnt[kMaxWorld];
    uint32_t* lastacc[kMaxWorld];
    const uint8_t* pool[kMaxWorld];
    const uint32_t* abort;                  // this rank's abort word (k_wait_flags timeout) or null
};
void launch_local_merge(int kmax, const Rec* ws, int parts, int64_t B, int topk, const int32_t* qstatus,
                        const uint32_t* present, int owner, cache_shard_rec* out, cudaStream_t s);
// recs[r][rec_row0 + i][topk] with row stride rec_stride (all-gathered lists: stride = B,
// rec_row0 = row0; the push inbox: stride = nb, rec_row0 = 0); inv_q / qstatus by global row
void launch_merge_sharded(int kmax, const cache_shard_rec* recs, int64_t rec_stride, int64_t rec_row0, int world,
                          int64_t row0, int64_t nb, int topk, const float* inv_q, const int32_t* qstatus,
                          const PeerPtrs& peers, uint32_t clock, int64_t latent_bytes, const KMap& km,
                          uint64_t* out_ids, float* out_scores, int32_t* out_k, uint8_t* latent_out, void** out_ptr,
                          int32_t* out_status, cudaStream_t s);

// ---- push exchange over peer memory (cache_push_*): producer kernels store their results
// straight into the consumers' arenas and the last CTA to finish publishes an epoch flag ----
struct PushSignal {
    uint32_t* flag[kMaxWorld];   // this sender's flag word in every rank's arena
    int world;
    uint32_t* done;              // local CTA-completion counter (zero between launches)
    uint32_t epoch;
    const uint32_t* abort;       // this rank's abort word: set once a peer wait timed out -> no more
                                 // stores into peer memory, no more publication
};
struct PushRows {                // destinations of the pushed query rows, one per rank
    __nv_bfloat16* y[kMaxWorld];
    float* inv[kMaxWorld];
    int32_t* status[kMaxWorld];
    int n;
};
struct PushRecs {                // record inbox of every rank: [sender][nb][topk]
    cache_shard_rec* inbox[kMaxWorld];
    int64_t nb;                  // rows owned per rank: global row q belongs to rank q / nb
    int me;
};
void launch_normalise_push(const void* x, int dtype, int64_t n, int dim, const PushRows& out, int64_t row0,
                           const PushSignal& sig, cudaStream_t s);
void launch_local_merge_push(int kmax, const Rec* ws, int parts, int64_t B, int topk, const int32_t* qstatus,
                             const uint32_t* present, int owner, const PushRecs& dst, const PushSignal& sig,
                             cudaStream_t s);
// Wait until every rank's flag reached `epoch`; a rank that has not published within
// timeout_ns (globaltimer) sets bit r of *abort (device) and *err_host (mapped host memory) and
// the wait returns, so the consumers behind it skip their peer accesses and the host reports
// CACHE_E_NCCL instead of the context dying (round 1: __trap) or the stream hanging.
void launch_wait_flags(const uint32_t* flags, int world, uint32_t epoch, unsigned long long timeout_ns,
                       uint32_t* abort, uint32_t* err_host, cudaStream_t s);
// Eviction histogram pass whose counts go straight into every rank's accumulator (P2P
// atomics) instead of a local buffer for an all-reduce; the grid then publishes `sig`.
struct PushHist {
    unsigned int* dst[kMaxWorld];
    int world;
};
void launch_push_hist_bins(const uint32_t* local, int nbins, const PushHist& ph, const PushSignal& sig, cudaStream_t s);
void launch_evict_hist_push(const uint32_t* present, const uint32_t* fcnt, const uint32_t* lastacc,
                            const uint32_t* ids, int64_t n_slots, const KMap& km, const EvictState* st, int pass,
                            const PushHist& ph, const PushSignal& sig, cudaStream_t s);

}  // namespace nv
