/*
 * nirvana_cache.h -- C ABI of the B200-native NIRVANA cache lookup (arXiv 2312.04429).
 *
 * The library implements the data-parallel hot path of the paper's approximate cache:
 * Alg. 1 lines 4-8 for a BATCH of prompt embeddings, plus the LCBFU
 * cache-maintenance calls.  Citations "P:n" are lines of the paper text
 * (/root/reference/PAPER.md); "R<n>" are the readings listed in DESIGN.md.
 *
 * Conventions (all calls):
 *   - Device memory: "device pointer" means a pointer returned by cudaMalloc on the cache's
 *     device (or managed memory).  "host pointer" means ordinary host memory (pinned memory
 *     is faster for the _host variants).  Every buffer is owned by the caller and must stay
 *     valid until the call's stream has passed it; the library copies what it keeps
 *     (embeddings, latents) into storage it owns.
 *   - Streams: `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Errors: every call returns a cache_status; argument and state errors are detected
 *     synchronously and leave the cache unchanged.  Asynchronous CUDA errors surface as
 *     CACHE_E_CUDA on a later call.  cache_last_error() gives a thread-local message.
 *   - Concurrency: one writer.  cache_insert / cache_evict must not overlap queries on the
 *     same handle (SPEC S:222's single-writer contract).
 *   - Ids: every stored prompt embedding (entry) gets an id = insertion sequence number
 *     (0, 1, 2, ...), used for deterministic tie-breaking (R3) and reported by queries.
 *   - Items: an item is one stored intermediate state (entry, K).
 */
#ifndef NIRVANA_CACHE_H
#define NIRVANA_CACHE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct cache_t cache_t; /* opaque handle, one per device (per rank) */

typedef enum {
    CACHE_OK = 0,
    CACHE_E_INVALID_ARG = 1, /* bad pointer / size / config value                          */
    CACHE_E_DIM = 2,         /* dim unsupported (must be a multiple of 64, <= 1024)         */
    CACHE_E_FULL = 3,        /* insert does not fit entry or latent capacity  */
    CACHE_E_EVICT_RANGE = 4, /* evict n > live items                          */
    CACHE_E_BAD_ROWS = 5,    /* some input rows rejected; per-row codes were written       */
    CACHE_E_CUDA = 6,        /* CUDA runtime/driver error                                  */
    CACHE_E_NCCL = 7,        /* a peer rank failed: a push-exchange wait timed out (dead or
                                stalled rank, cache_set_peer_timeout), or (binding) an NCCL
                                collective of the sharded protocol failed                   */
    CACHE_E_OOM = 8,         /* device allocation failed                                   */
    CACHE_E_STATE = 9,       /* call not valid in the handle's state (e.g. id space spent) */
    CACHE_E_UNSUPPORTED = 10 /* requested variant not built for this configuration         */
} cache_status;

/* per-row status codes (row_status outputs) */
enum {
    CACHE_ROW_OK = 0,
    CACHE_ROW_NONFINITE = 1, /* a component is NaN/Inf                 */
    CACHE_ROW_ZERO_NORM = 2, /* zero vector: "degenerate embedding"      */
    CACHE_ROW_NO_ITEMS = 3   /* insert: present mask selects no K, nothing to store */
};

/* input element types of embeddings / queries */
enum { CACHE_DTYPE_F32 = 0, CACHE_DTYPE_BF16 = 1 };

/* scoring kernel selection (cache_set_scorer) */
enum {
    CACHE_SCORER_AUTO = 0,   /* library picks by batch size                                */
    CACHE_SCORER_TC = 1,     /* tcgen05/TMEM tensor-core scan with fused top-k epilogue    */
    CACHE_SCORER_STREAM = 2, /* CUDA-core HBM-streaming scan (small batches)               */
    CACHE_SCORER_TC_SINGLE = 3 /* tcgen05 scan with single-CTA tiles only (no CTA pairs);
                                  AUTO / TC use CTA pairs (cta_group::2) when b > 128       */
};

#define CACHE_MAX_K 8      /* max |K| (the paper uses 5: {5,10,15,20,25})           */
#define CACHE_MAX_TOPK 16  /* max m nearest neighbours returned per query           */
#define CACHE_NO_ID UINT64_MAX

typedef struct {
    int32_t dim;              /* embedding dimension; 768 for CLIP; multiple of 64  */
    int64_t entry_capacity;   /* max live entries (prompt embeddings)                      */
    int64_t latent_capacity;  /* max live items (latent-pool slots); decoupled from entries
                                 as in "1.5 million intermediate-states ... 300k unique
                                 prompt embedding"                                 */
    int64_t latent_bytes;     /* bytes per stored intermediate state, opaque; multiple of 16
                                 (144 KB in the paper P:511; 4x64x64 fp16 = 32768 here)    */
    int32_t num_k;            /* |K| <= CACHE_MAX_K                                        */
    int32_t k_values[CACHE_MAX_K];   /* K values, strictly increasing ({5,..,25})   */
    double thresholds[CACHE_MAX_K];  /* Fig. 11: K = k_values[j] for the largest
                                        j with s > thresholds[j] (strict), else 0; must be
                                        non-decreasing ({.65,.75,.85,.90,.95})              */
    int32_t k_bias;           /* quality-vs-savings knob (R20): on a hit the
                                 bucket moves up by k_bias (clamped); 0 = Fig. 11 verbatim */
    int32_t max_topk;         /* largest topk a query may request (<= CACHE_MAX_TOPK)      */
    int32_t shard_rank;       /* entry sharding over shard_world GPUs: every  */
    int32_t shard_world;      /* rank receives the same insert batches; accepted rows get
                                 global ids 0,1,2,... and rank r stores the rows with
                                 id % shard_world == r.  Default 0 / 1 = unsharded.         */
    int32_t latent_alias;     /* 0: every stored (entry, K) owns a pool slot (default).
                                 1: declared aliasing for caches whose full per-K state
                                 store exceeds HBM: item (id, j) reads
                                 pool slot CACHE_ALIAS_SLOT(id, j, latent_capacity); inserts
                                 take no payload (latents must be NULL) and consume no pool
                                 capacity; the pool is filled with cache_pool_write and is
                                 never freed by eviction.                                  */
    int32_t evict_policy;     /* CACHE_POLICY_*: which item score cache_evict minimises     */
    int32_t evict_granularity; /* CACHE_EVICT_ITEM (default, the paper's) or CACHE_EVICT_ENTRY */
} cache_config;

/* Eviction granularity (SURVEY 8(b) / reading c10, DESIGN R24).
 * ITEM:  cache_evict(n) removes the n (entry, K) items with the smallest policy score
 *        (P:602-611); entries left with no K are dirty and removed too.
 * ENTRY: cache_evict(n) removes n whole entries, those with the smallest ENTRY score = the
 *        policy score aggregated over the entry's stored items -- LCBFU sum f_j x K_j (the
 *        segmented reduction), LFU sum f_j, LRU max of the items' last-access clocks, FIFO 0 --
 *        ties by id ascending; every stored state of an evicted entry is freed. */
enum { CACHE_EVICT_ITEM = 0, CACHE_EVICT_ENTRY = 1 };

/* Eviction policies: the item score minimised by cache_evict (ties by (id, K) ascending).
 * LCBFU is the paper's policy; the others are the baselines it is compared with. */
enum {
    CACHE_POLICY_LCBFU = 0, /* f_i x K_i: access frequency x computation saved   */
    CACHE_POLICY_LRU = 1,   /* batch clock of the last access; insert clock until accessed
                                                                       */
    CACHE_POLICY_LFU = 2,   /* f_i                                               */
    CACHE_POLICY_FIFO = 3   /* insertion order: the id alone                     */
};

/* The declared aliasing map of latent_alias = 1 (a plain, documented function of the id). */
#define CACHE_ALIAS_SLOT(id, j, cap) \
    ((int64_t)(((uint32_t)(id) * 8u + (uint32_t)(j)) * 2654435761u) % (int64_t)(cap))

typedef struct {
    int64_t live_entries;     /* prompt embeddings present in the index                   */
    int64_t live_items;       /* stored (entry, K) intermediate states                    */
    int64_t holes;            /* missing K among live entries                     */
    int64_t entry_hwm;        /* high-water mark of entry slots (the scan length)          */
    uint64_t next_id;         /* id the next inserted entry receives                       */
    int64_t queries;          /* queries answered so far                                   */
    int64_t free_entries;     /* free entry slots on this rank                              */
    int64_t free_items;       /* free latent-pool slots on this rank                        */
} cache_stats_t;

/* One partial top-k record of a shard (16 bytes): the ranking key of an entry,
 * key = orderable_f32(t) << 32 | (2^32 - 1 - id) with t = fl(<q~,x~> * inv_norm(x~)) (a larger
 * key is a better candidate, 0 = none), the entry's slot and presence mask on its owner rank. */
typedef struct {
    uint64_t key;
    uint32_t slot;
    uint8_t present_mask;
    uint8_t owner;
    uint16_t reserved;
} cache_shard_rec;

/* Radix-select state of a (possibly distributed) LCBFU eviction; lives in device memory. */
typedef struct {
    uint64_t prefix;     /* selected high digits of the n-th smallest item key so far  */
    uint64_t mask;       /* which digits of prefix are decided                         */
    uint64_t remaining;  /* rank of the target key among keys matching prefix (1-based) */
} cache_evict_state;

/* What a rank shares with its peers so their merge kernels can read its latent pool and
 * slot tables and count accesses on its counters directly over NVLink (P2P loads/atomics). */
typedef struct {
    int32_t device;
    int32_t pid;
    int32_t num_k;
    int32_t reserved;
    int64_t latent_bytes;
    void *lslot, *fcnt, *pool, *lastacc;           /* raw device pointers (same process)   */
    unsigned char ipc_lslot[64], ipc_fcnt[64], ipc_pool[64], ipc_lastacc[64]; /* IPC handles */
    void *arena;                 /* push-exchange arena (cache_push_reserve) or NULL          */
    int64_t arena_nb;            /* its geometry: max local batch, max topk                   */
    int32_t arena_topk;
    int32_t reserved2;
    unsigned char ipc_arena[64];
    uint64_t process_token;      /* random per-process identity: raw pointers are used only when
                                    pid AND token match (PID namespaces can repeat pids)      */
} cache_peer_desc;

/* Fill *cfg with the paper's defaults: dim 768, K = {5,10,15,20,25}, Fig. 11
 * thresholds, k_bias 0, max_topk 16, latent_bytes 32768. Capacities are set to 0
 * and must be filled in by the caller. */
void cache_default_config(cache_config *cfg);

/* Create a cache on CUDA device `device`, allocating all storage up front (HBM footprint
 * ~ entry_capacity*(2*dim + 4*(2+2*num_k)) + latent_capacity*latent_bytes bytes).
 * Host-synchronous.  *out receives the handle. */
cache_status cache_create(const cache_config *cfg, int device, cache_t **out);

/* Free all storage.  Synchronises the device.  NULL is a no-op. */
cache_status cache_destroy(cache_t *c);

/* LCBFU insertion: store n prompt embeddings and their intermediate states.
 *   emb        device pointer, n x dim row-major, element type emb_dtype (CACHE_DTYPE_*)
 *   latents    device pointer, n x num_k x latent_bytes (state of row r at K_j at
 *              ((r*num_k)+j)*latent_bytes), or NULL to store no payload bytes
 *   present    device or host pointer, n bitmasks (bit j set = K_j is stored), or NULL = all
 *   out_ids    host pointer, n ids (CACHE_NO_ID for a rejected row); may be NULL
 *   row_status host pointer, n CACHE_ROW_* codes; may be NULL
 * Each accepted row is normalised in fp64 (sum of squares in a fixed halving-tree order,
 * correctly rounded sqrt and division) and rounded to bf16 (RNE) -- reading R2: a stored
 * component can differ from the plain index-order definition only where the exact quotient
 * lies within the two summation orders' fp64 error bound of a bf16 rounding midpoint.  Rows with
 * non-finite components or zero norm are rejected (CACHE_E_BAD_ROWS after the valid rows
 * are stored).  If the accepted rows exceed the free entry or latent capacity the call
 * returns CACHE_E_FULL and stores nothing (no automatic eviction, R14).
 * Synchronises `stream` (slot allocation needs the row statuses). */
cache_status cache_insert(cache_t *c, int64_t n, const void *emb, int32_t emb_dtype,
                          const void *latents, const uint8_t *present, uint64_t *out_ids,
                          int32_t *row_status, void *stream);

/* Batched cache lookup: Alg. 1 lines 4-8 for b queries at once.
 *   queries        device pointer, b x dim, element type q_dtype
 *   topk           1..max_topk nearest cached entries to report
 *   out_ids        device pointer, b x topk u64: entry ids by (score desc, id asc);
 *                  CACHE_NO_ID where fewer than topk live entries exist
 *   out_scores     device pointer, b x topk f32 cosine similarities clamped to [-1,1]
 *                  (-inf where no entry); ranking uses the unclamped value (R4)
 *   out_k          device pointer, b i32: K used for query i after the Fig. 11 map
 *                   and the hole rule; 0 = generate from scratch
 *   latent_out     device pointer, b x latent_bytes: row i receives the stored state
 *                  (entry top-1, K = out_k[i]) iff out_k[i] > 0; other rows are
 *                  not written.  May be NULL (no gather).
 *   out_latent_ptr device pointer, b void*: &latent_out[i*latent_bytes] or NULL; may be NULL
 *   row_status     device pointer, b i32 CACHE_ROW_*; may be NULL
 * For every query with out_k[i] > 0 the LCBFU access count f[(entry, K)] is incremented by
 * one after the batch (R8/R9).  Asynchronous on `stream`; returns after launch.
 * Cosine similarity is computed exactly over every live entry (R1) on the stored bf16
 * values with fp32 accumulation: s = fl(fl(<q~,x~> * inv_norm(x~)) * inv_norm(q~)). */
cache_status cache_query_batch(cache_t *c, int64_t b, const void *queries, int32_t q_dtype,
                               int32_t topk, uint64_t *out_ids, float *out_scores,
                               int32_t *out_k, void *latent_out, void **out_latent_ptr,
                               int32_t *row_status, void *stream);

/* Read-only batched lookup: the ids, scores and K that cache_query_batch would report for the
 * same cache state, but NO access is counted (no LCBFU counter, no LRU clock tick) and no
 * state is gathered.  For measurements that must not disturb the eviction state: the match
 * predictor's would-hit statistics of requests it sends to scratch generation (Alg. 1 line 2,
 * a predicted miss performs no search), and profiling.  Buffers as cache_query_batch
 * (device pointers); asynchronous on `stream`. */
cache_status cache_query_peek(cache_t *c, int64_t b, const void *queries, int32_t q_dtype, int32_t topk,
                              uint64_t *out_ids, float *out_scores, int32_t *out_k, int32_t *row_status,
                              void *stream);

/* Same lookup called from the host (the end-to-end call a serving process makes): queries,
 * out_ids, out_scores, out_k and row_status are host pointers (pinned memory recommended);
 * the library copies the queries in, runs the lookup, copies ids/scores/K/status back in one
 * transfer and synchronises `stream` before returning.  latent_out may be a DEVICE pointer
 * (the denoiser's input buffer on this GPU: states are gathered there directly, nothing
 * crosses PCIe) or a HOST pointer (staged on the device, then copied back); it may be NULL.
 * row_status may be NULL. */
cache_status cache_query_batch_host(cache_t *c, int64_t b, const void *queries, int32_t q_dtype,
                                    int32_t topk, uint64_t *out_ids, float *out_scores,
                                    int32_t *out_k, void *latent_out, int32_t *row_status,
                                    void *stream);

/* Pipelined host calls (two slots): cache_query_submit enqueues one batch -- the upload of
 * `queries` (HOST memory, pinned for overlap; must stay valid until the slot completes) on the
 * library's copy stream, the lookup of cache_query_batch on `stream` once it has landed, the
 * download of the results into pinned staging -- and returns at once; cache_query_complete
 * waits for that slot and copies ids / scores / K / status to the caller's host arrays.  While
 * slot i's lookup runs, slot i^1's upload proceeds, so a loop
 *     submit(0, q0); submit(1, q1); complete(0); submit(0, q2); complete(1); ...
 * overlaps each batch's host-to-device copy with the previous batch's scan (the synchronous
 * cache_query_batch_host cannot).  latent_out: DEVICE pointer (the denoiser's input buffer for
 * this batch) or NULL.  One LRU clock tick per submitted batch; batches run in submit order.
 * CACHE_E_STATE: submit on a pending slot / complete on an idle one. */
cache_status cache_query_submit(cache_t *c, int32_t slot, int64_t b, const void *queries, int32_t q_dtype,
                                int32_t topk, void *latent_out, void *stream);
cache_status cache_query_complete(cache_t *c, int32_t slot, uint64_t *out_ids, float *out_scores,
                                  int32_t *out_k, int32_t *row_status);

/* LCBFU eviction: remove the n stored items with the smallest LCBFU score
 * f_i x K_i, ties by (entry id, K) ascending (R11); then every entry left with no
 * stored K is dirty and is removed from the index in the same call (R13).
 *   out_evicted    host pointer, n u64 (id << 3 | j) in eviction order; may be NULL
 *   out_dirty_ids  host pointer, capacity n, ids of removed entries ascending; may be NULL
 *   out_n_dirty    host pointer, number of entries removed; may be NULL
 * n > live items -> CACHE_E_EVICT_RANGE.  Synchronises `stream`.
 * With evict_granularity = CACHE_EVICT_ENTRY, n counts entries (n > live entries ->
 * CACHE_E_EVICT_RANGE), out_evicted receives the n entry ids in eviction order (ascending
 * entry score, then id) and out_dirty_ids the same ids ascending (*out_n_dirty = n). */
cache_status cache_evict(cache_t *c, int64_t n, uint64_t *out_evicted, uint64_t *out_dirty_ids,
                         int64_t *out_n_dirty, void *stream);
/* cache_evict without the copies into caller memory: on success *out_evicted (n values, as
 * cache_evict's out_evicted) and *out_dirty_ids (*out_n_dirty ids, ascending) point into the
 * library's pinned staging of this handle, valid until its next eviction or destroy (a serving
 * loop consumes them at once; copying 5 MB of lists per 1% eviction at 12.5M entries cost more
 * host time than the GPU work). */
cache_status cache_evict_view(cache_t *c, int64_t n, const uint64_t **out_evicted,
                              const uint64_t **out_dirty_ids, int64_t *out_n_dirty, void *stream);

/* The full 64-bit unit keys (R11 / R24: score << 35 | id << 3 | j, or score << 32 | id) of the
 * last cache_evict / cache_evict_apply / cache_push_evict_apply that returned its evicted list,
 * in eviction order (ascending).  Lets a sharded caller merge the ranks' lists into the global
 * eviction order.  out: host array of capacity cap; *out_n = the number of keys available. */
cache_status cache_last_evicted_keys(cache_t *c, uint64_t *out, int64_t cap, int64_t *out_n);

/* ---- distributed eviction building blocks (cache_evict = these three with no exchange) ----
 * The n lowest LCBFU keys across all shards are found by an 8-pass MSB-first radix select
 * over 8-bit digits of the 64-bit item key (R11).  Per pass: cache_evict_hist computes this
 * rank's 256-bin histogram of keys matching st->prefix (hist: device, 256 u32, overwritten);
 * the caller sums the histograms over ranks (e.g. an NCCL all-reduce); cache_evict_pick then
 * fixes the pass's digit in st (identically on every rank).  st starts as {0, 0, n}.
 * cache_evict_apply evicts this rank's items with key <= st->prefix (the n-th smallest key)
 * and removes its dirty entries.  Outputs are host arrays of capacity `cap`: evicted items
 * (id << 3 | j) in key order, removed entry ids ascending; counts in *out_n / *out_n_dirty.
 * out_evicted and/or out_dirty_ids may be NULL: that list is then neither sorted nor copied
 * (the counts are still reported).  Synchronises `stream`. */
cache_status cache_evict_hist(cache_t *c, const cache_evict_state *st, int32_t pass,
                              uint32_t *hist, void *stream);
cache_status cache_evict_pick(cache_t *c, uint32_t *hist, cache_evict_state *st, int32_t pass,
                              void *stream);
cache_status cache_evict_apply(cache_t *c, const cache_evict_state *st, int64_t cap,
                               uint64_t *out_evicted, int64_t *out_n, uint64_t *out_dirty_ids,
                               int64_t *out_n_dirty, void *stream);
/* Live items on this rank (host-synchronous). */
int64_t cache_live_items(const cache_t *c);
/* Live entries on this rank (host-synchronous). */
int64_t cache_live_entries(const cache_t *c);

/* ---- sharded lookup ----
 * 1. every rank gathers the global batch of b queries (caller's all-gather);
 * 2. cache_query_local: ingest + tcgen05 scan of this rank's shard + local top-k ->
 *    out_recs (device, b x topk cache_shard_rec, owner = shard_rank);
 * 3. the caller all-gathers the records of all ranks -> recs (device, world x b x topk);
 * 4. cache_query_merge: for global rows [row0, row0 + nb) merge the world lists under the
 *    total order (R3), apply Fig. 11 + holes, copy the winning state straight from the
 *    owner's latent pool (P2P over NVLink) into latent_out and count the access on the
 *    owner's counters (P2P atomics).  Outputs as in cache_query_batch, nb rows each.
 * cache_attach_peers must have been called with every rank's cache_export_peer(). */
cache_status cache_query_local(cache_t *c, int64_t b, const void *queries, int32_t q_dtype,
                               int32_t topk, cache_shard_rec *out_recs, void *stream);
cache_status cache_query_merge(cache_t *c, int64_t b, int64_t row0, int64_t nb, int32_t topk,
                               const cache_shard_rec *recs, uint64_t *out_ids, float *out_scores,
                               int32_t *out_k, void *latent_out, void **out_latent_ptr,
                               int32_t *row_status, void *stream);
cache_status cache_export_peer(cache_t *c, cache_peer_desc *out);
cache_status cache_attach_peers(cache_t *c, int32_t world, const cache_peer_desc *descs);

/* ---- sharded lookup with the exchanges fused into the kernels (SURVEY 8(e) "fusing the
 * record push"; no collective library on the data path) ----
 * Every rank owns an exchange ARENA in its HBM (flags, the global query batch as bf16 rows +
 * inv-norms + statuses, and a record inbox); peers write into it over NVLink (P2P stores
 * through CUDA IPC mappings).  Rank r's local batch is global rows [r*nb, r*nb + nb).
 *  cache_push_reserve  allocate the arena for local batches <= max_nb and topk <= max_topk;
 *                      call before cache_export_peer (the descriptor carries its IPC handle).
 *  phase 1  cache_push_queries: ingest this rank's nb queries (the a1 rule) and store each
 *           normalised row straight into EVERY rank's arena (the query all-gather fused
 *           into the ingest kernel); the grid's last CTA publishes the batch epoch on every
 *           rank's query flag for this sender (st.release.sys).
 *  phase 2  cache_push_scan: wait for all ranks' query flags (ld.acquire.sys), tcgen05 scan
 *           of this rank's shard for all world*nb rows, then the local merge stores each
 *           row's top-k shard records straight into the OWNER's inbox (the record exchange
 *           fused into the merge kernel) and publishes the epoch on the record flags.
 *  phase 3  cache_push_merge: wait for all ranks' record flags, then merge this rank's own
 *           rows exactly as cache_query_merge (P2P latent fetch, P2P counter atomics).
 * Every rank calls the three phases in order, once per batch, with the same nb and topk
 * (ranks in separate processes may call them back to back; virtual ranks in one process on
 * one stream call phase 1 on all ranks, then phase 2, then phase 3).  Outputs as in
 * cache_query_batch, nb rows.  Arena reuse across batches needs no extra barrier: a rank
 * writes batch t+1 into a peer's arena only after the peer has published batch t+1's queries,
 * i.e. after it finished merging batch t.
 * Failure (failure detection): a wait that sees no progress from some rank within
 * the peer timeout (default 10 s; cache_set_peer_timeout, or NIRVANA_PEER_TIMEOUT_MS at
 * create) marks the handle failed instead of hanging or trapping: the kernels behind it skip
 * every peer load / store, the CUDA context stays usable, and every later cache_push_* call
 * (and cache_push_status, which synchronises `stream` first) returns CACHE_E_NCCL.  The
 * outputs of the failed batch are undefined; local (unsharded) calls keep working. */
cache_status cache_push_reserve(cache_t *c, int64_t max_nb, int32_t max_topk);
/* Synchronise `stream`, then CACHE_E_NCCL if a peer wait of this handle timed out, else OK. */
cache_status cache_push_status(cache_t *c, void *stream);
/* Peer timeout of the push-exchange waits (ms > 0). */
cache_status cache_set_peer_timeout(cache_t *c, int64_t timeout_ms);
cache_status cache_push_queries(cache_t *c, int64_t nb, const void *queries, int32_t q_dtype, void *stream);
cache_status cache_push_scan(cache_t *c, int64_t nb, int32_t topk, void *stream);
cache_status cache_push_merge(cache_t *c, int64_t nb, int32_t topk, uint64_t *out_ids, float *out_scores,
                              int32_t *out_k, void *latent_out, void **out_latent_ptr, int32_t *row_status,
                              void *stream);

/* Distributed FUSED eviction (round 2; replaces the 8-pass radix protocol above for sharded
 * caches): cache_evict's single-launch algorithm cut at its histogram exchanges -- level 0 a
 * sweep of this shard into 4,096 log bins, levels >= 1 a sweep that applies the units certain
 * to go and compacts the chosen range's candidates (later levels sweep only those), every
 * level's histogram summed over ranks before every rank takes the same pick; then the final
 * apply and the ordered lists.  Typically 2 sweeps of the slot columns instead of 9.
 * Collective, every rank with the same n (the GLOBAL number of units to evict):
 *   cache_evict_sel_begin(c, n)
 *   for level = 0, 1, ...:
 *     cache_evict_sel_level(c, level, hist)     hist: device u32[4096], this rank's histogram
 *     (sum hist over the ranks, e.g. an NCCL all-reduce)
 *     cache_evict_sel_pick(c, level, hist_sum, &done)   host-synchronous; stop when done != 0
 *   cache_evict_sel_apply(c, cap, ...)          outputs as cache_evict_apply (this rank's share)
 * or, with the push arenas (cache_push_reserve), the exchange over peer memory instead:
 *   cache_push_evict_sel_level(c, level); cache_push_evict_sel_pick(c, level, &done)
 * (virtual ranks in one process: level on every rank, then pick on every rank).  Every rank
 * runs the same number of levels (the picks agree).  Errors: CACHE_E_STATE out of order. */
cache_status cache_evict_sel_begin(cache_t *c, int64_t n, void *stream);
cache_status cache_evict_sel_level(cache_t *c, int32_t level, uint32_t *hist, void *stream);
cache_status cache_evict_sel_pick(cache_t *c, int32_t level, const uint32_t *hist_sum, int32_t *out_done,
                                  void *stream);
cache_status cache_evict_sel_apply(cache_t *c, int64_t cap, uint64_t *out_evicted, int64_t *out_n,
                                   uint64_t *out_dirty_ids, int64_t *out_n_dirty, void *stream);
cache_status cache_push_evict_sel_level(cache_t *c, int32_t level, void *stream);
cache_status cache_push_evict_sel_pick(cache_t *c, int32_t level, int32_t *out_done, void *stream);

/* Fused distributed eviction (the radix-select histograms of cache_evict_hist / _pick without
 * a collective): pass p's histogram kernel adds its counts straight into EVERY rank's arena
 * accumulator (P2P atomics over NVLink) and publishes a per-pass epoch flag; the pick waits
 * for all ranks' flags, reads the complete global histogram from its own arena and fixes the
 * pass's digit (identically on every rank).  Collective: every rank calls, with the same n,
 *   for p in 0..7: cache_push_evict_hist(c, n, p); cache_push_evict_pick(c, p);
 *   then cache_push_evict_apply(c, n, ...)  (outputs as cache_evict_apply, capacity n)
 * (virtual ranks in one process: hist(p) on all ranks, then pick(p) on all ranks).  The
 * selection state lives in the cache.  Needs cache_push_reserve on every rank (the arena). */
cache_status cache_push_evict_hist(cache_t *c, int64_t n, int32_t pass, void *stream);
cache_status cache_push_evict_pick(cache_t *c, int32_t pass, void *stream);
cache_status cache_push_evict_apply(cache_t *c, int64_t n, uint64_t *out_evicted, int64_t *out_n,
                                    uint64_t *out_dirty_ids, int64_t *out_n_dirty, void *stream);

/* ---- cache-selector profiling (Alg. 2) ----
 * "generates images at each value of K for a set of prompts with their nearest cache prompt.
 * It then finds the minimum similarity score such that all generated images are above a
 * quality threshold alpha".  The images and their quality come from the diffusion
 * model (outside this library): the caller passes quality[j*b + i] = the quality reached by
 * profiling prompt i when reconditioning its nearest cached prompt's state at K = k_values[j]
 * (device pointer, num_k x b floats).  The library computes the prompt's similarity to its
 * nearest cached entry with the exact top-1 scan (as cache_query_batch scores it; no access is
 * counted) and, reading R25, returns per K the largest similarity at which some profiled
 * image failed (quality <= alpha) -- so every profiled pair with s > threshold passed, matching
 * the strict '>' of Fig. 11 -- or, if none failed, the smallest profiled similarity;
 * thresholds are made non-decreasing in K.  out_thresholds: host, num_k doubles;
 * out_failed: host, num_k int64 (1 if some pair failed at that K) or NULL.  Host-synchronous.
 * cache_set_thresholds installs a table (non-decreasing) for later lookups. */
cache_status cache_profile_thresholds(cache_t *c, int64_t b, const void *queries, int32_t q_dtype,
                                      const float *quality, double alpha, double *out_thresholds,
                                      int64_t *out_failed, void *stream);
cache_status cache_set_thresholds(cache_t *c, const double *thresholds);

/* ---- match predictor ----
 * A linear one-class SVM f(x) = <w, x> - rho over the cached embeddings (unit-scaled stored
 * values), "trained by utilizing all prompt embeddings stored in the VDB" with
 * nu (0.001 in the paper).  Training (reading R22): rho is set each epoch to the
 * ceil(nu n)-th smallest margin (the exact minimiser of the one-class objective in rho) and w
 * takes a subgradient step w <- w - eta_t (nu w - (1/n) sum_{<w,x_i> < rho} x_i) / nu with
 * eta_t = lr0 / sqrt(1 + t), from w = mean(x_i); `epochs` steps.  Synchronises `stream`.
 * cache_predict: out_flags[i] = 1 iff f(q~_i / ||q~_i||) >= 0 ("a close match is likely",
 * P:465-468), out_margin[i] = f (device pointers; either may be NULL; rejected rows get 0 /
 * -inf).  Asynchronous.  cache_predictor_get copies w (dim floats) and rho to the host. */
cache_status cache_predictor_train(cache_t *c, double nu, int32_t epochs, double lr0, void *stream);
cache_status cache_predict(cache_t *c, int64_t b, const void *queries, int32_t q_dtype,
                           uint8_t *out_flags, float *out_margin, void *stream);
cache_status cache_predictor_get(cache_t *c, float *w, float *rho);

/* Write n consecutive latent-pool slots starting at slot0 from `src` (device pointer,
 * n x latent_bytes).  Asynchronous.  Used to pre-fill an aliased pool (latent_alias = 1). */
cache_status cache_pool_write(cache_t *c, int64_t slot0, int64_t n, const void *src, void *stream);

/* Counters: read the LCBFU access counts and presence mask of entry `id` (host outputs,
 * f has num_k slots).  Host-synchronous; intended for tests and maintenance tools. */
cache_status cache_get_meta(cache_t *c, uint64_t id, uint64_t *f, uint32_t *present_mask);

/* Copy the stored bf16 row of entry `id` to host memory (dim uint16 bit patterns). */
cache_status cache_get_row(cache_t *c, uint64_t id, uint16_t *out_bf16);

/* Host-synchronous statistics. */
cache_status cache_stats(cache_t *c, cache_stats_t *out);

/* The handle's live configuration: cache_create's, with the threshold table, k_bias, policy and
 * granularity as later calls set them (cache_set_thresholds / _evict_policy / _granularity).
 * *out is caller-owned. */
cache_status cache_get_config(cache_t *c, cache_config *out);

/* Checkpoint / resume (the paper's cache persists as EFS files + a Qdrant collection,
 * P:508-511).  cache_save writes the handle's whole state to the file `path`: the live
 * configuration, the stored bf16 rows and inverse norms, ids, presence masks, latent-pool slots,
 * LCBFU counters and LRU clocks of slots [0, high-water mark), the host allocator state (entry /
 * pool free lists, next id, LRU batch clock, query count), the trained match predictor if any,
 * and -- with_latents != 0 -- the occupied prefix of the latent pool (aliased pools: all of it).
 * cache_load creates a handle on `device` holding exactly that state: every later call answers
 * as the saved handle would have (tested bit for bit).  A shard saves its own state; push
 * arenas and peer mappings are not saved (re-run cache_push_reserve / cache_attach_peers).
 * Host-synchronous; the file is this library version's layout (magic + version checked).
 * Errors: CACHE_E_INVALID_ARG (null, file not writable / readable, foreign or truncated file),
 * CACHE_E_OOM / CACHE_E_CUDA (device allocation or copies); *out is NULL on failure. */
cache_status cache_save(cache_t *c, const char *path, int32_t with_latents);
cache_status cache_load(const char *path, int32_t device, cache_t **out);

/* Select the eviction policy (CACHE_POLICY_*) used by later cache_evict calls. */
cache_status cache_set_evict_policy(cache_t *c, int32_t policy);
/* Select the eviction granularity (CACHE_EVICT_ITEM / CACHE_EVICT_ENTRY) of later evictions. */
cache_status cache_set_evict_granularity(cache_t *c, int32_t granularity);

/* Force a scoring kernel (CACHE_SCORER_*); AUTO by default. */
cache_status cache_set_scorer(cache_t *c, int32_t scorer);

/* Query slicing of cache_query_batch (a scheduling choice; results are identical for every
 * value -- each query's answer depends only on its own row and the pre-batch state, R9).
 * With n > 1 slices the tensor-core scan runs as n launches over consecutive query slices of
 * a multiple of 256 rows, and slice i's finalize + latent gather (a1-a8's HBM-bound tail,
 * P:434-435) runs on a library-owned side stream concurrently with slice i+1's scan; the call's
 * stream waits for all of them before later work.  0 = auto (currently one launch: at C2 the
 * concurrent finalize slows the scan by more than the gather it hides),
 * 1 = never, 2..8 = that many slices (batches of more than 256 queries).
 * CACHE_E_INVALID_ARG outside [0, 8]. */
cache_status cache_set_query_slices(cache_t *c, int32_t slices);

/* Profiling hook: `events` points to 4 cudaEvent_t handles (host array, or NULL to disable).
 * When set, every cache_query_batch records events[0] before query ingest, events[1] before
 * the scoring kernel, events[2] before the finalize/gather kernel and events[3] after it, on
 * the call's stream, so a caller can time each kernel with cudaEventElapsedTime.  With query
 * slices (cache_set_query_slices) events[1]..events[2] span every slice's scan (the side-stream
 * finalizes of the earlier slices run inside that span) and events[2]..events[3] the last
 * slice's finalize. */
cache_status cache_set_profile_events(cache_t *c, void *const *events);

/* Number of kernels the library launched on this handle so far (for launch accounting). */
int64_t cache_kernel_launches(const cache_t *c);

/* Thread-local description of the last error (never NULL). */
const char *cache_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* NIRVANA_CACHE_H */
