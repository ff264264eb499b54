/*
 * nirvana_oracle.c -- plain, slow, obviously-correct fp64 CPU oracle of the NIRVANA
 * per-request cache lookup (arXiv 2312.04429).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2312_04429_b200/) never links, imports or executes anything under oracle/,
 * and the two share no code, no header and no constant generator.
 *
 * What it computes, and where the paper defines it (P:n = /root/reference/PAPER.md line n):
 *   - insert      : LCBFU insertion of all |K| intermediate states of a prompt (P:606-609,
 *                   "Insertion"), the prompt embedding e_p stored after
 *                   normalisation + bf16 rounding (reading R2).
 *   - query       : Alg. 1 lines 4-8: search_VDB = nearest cached embedding by
 *                   cosine similarity, exact over every live entry (reading R1);
 *                   heuristics_K = Fig. 11 cache_selector (strict '>'), optional
 *                   knob (reading R20); hole rule "largest value K that is less than
 *                   or equal to the optimal K"; payload['noise'][K] retrieval
 *                   (P:434-435); LCBFU access frequency f_i.
 *   - evict       : LCBFU score f_i x K_i, "evict the top-|K| items from the heap
 *                   root" generalised to n (reading R12), dirty-prompt removal when all
 *                   K are holes.
 *
 * Arithmetic: IEEE fp64, every sum in plain index order, compiled with -ffp-contract=off
 * (no FMA contraction) and without -ffast-math.  No blocking, fusion or reordering.
 *
 * Parity pins (tests/test_oracle_pins.py): bf16 rounding vs spot values + an independent
 * bit-level rounding + torch's fp32->bf16 RNE; cosine vs 60-digit Decimal arithmetic and the
 * hand-worked exact cache H; K map vs Fig. 11's truth table; holes vs the paper/SPEC cases;
 * LCBFU order vs the paper's 2500/1000 example and brute-force optimality.
 */
#include <fenv.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_E_INVALID_ARG 1
#define ORC_E_FULL 3
#define ORC_E_EVICT_RANGE 4
#define ORC_E_BAD_ROWS 5
#define ORC_E_OOM 8

#define ORC_ROW_OK 0
#define ORC_ROW_NONFINITE 1
#define ORC_ROW_ZERO_NORM 2
#define ORC_ROW_NO_ITEMS 3   /* present mask selects no K: nothing to store */

#define ORC_MAX_K 8
#define ORC_NO_ID UINT64_MAX

typedef struct {
    uint64_t id;          /* insertion sequence number */
    int live;
    double *x;            /* fp64 values of the STORED bf16 components */
    double nrm;           /* sqrt(sum x_i^2), index order */
    int present[ORC_MAX_K];
    uint64_t f[ORC_MAX_K];            /* LCBFU access frequency per K */
    uint64_t last[ORC_MAX_K];         /* batch clock of the last access (LRU), insert clock at first */
    unsigned char *lat[ORC_MAX_K];    /* stored latent bytes per present K, or NULL (no payload) */
} oentry;

typedef struct {
    int dim;
    int64_t entry_capacity;
    int64_t latent_capacity;
    int64_t latent_bytes;
    int num_k;
    int k_values[ORC_MAX_K];
    double thresholds[ORC_MAX_K];
    int k_bias;
    oentry *e;            /* all entries ever inserted, in insertion (= id) order */
    int64_t n_e, cap_e;
    int64_t live_entries;
    int64_t live_items;
    uint64_t next_id;
    uint64_t clock;       /* number of query batches so far (the LRU logical clock) */
} oracle_cache;

/* ---------------------------------------------------------------------------------------
 * bf16 round-to-nearest-even of a double, done plainly: v = f * 2^e with 0.5 <= |f| < 1;
 * bf16 keeps 8 significant bits, so the rounding quantum is 2^(e-8), floored at the bf16
 * subnormal quantum 2^-133 (e clamped at -125).  Scaling by a power of two is exact in fp64
 * and nearbyint() rounds to nearest-even under the default rounding mode.
 * (Reading R2: stored embeddings are bf16, normalised in fp64 first.)
 * ------------------------------------------------------------------------------------- */
double oracle_bf16_round(double v)
{
    int e;
    double r;
    if (v == 0.0 || !isfinite(v)) return v;
    frexp(v, &e);
    if (e < -125) e = -125;
    r = nearbyint(ldexp(v, 8 - e));
    return ldexp(r, e - 8);
}

/* Sum of squares in plain index order, fp64, no FMA contraction: the definition of the norm
 * (SPEC S:53-56 `normalize`).  For fp32 or bf16 inputs every square is
 * exact in fp64, so only the 767 additions round, in the order i = 0, 1, ..., dim-1. */
static double sum_sq(const double *x, int dim)
{
    double s = 0.0;
    int i;
    for (i = 0; i < dim; i++) s = s + x[i] * x[i];
    return s;
}

/* Normalise one row: nu = sqrt(sum_i x_i^2) (fp64, index order above); y_i = bf16(x_i / nu).
 * Returns the row status (non-finite input or zero norm are rejected). */
static int normalise_row(const double *x, int dim, double *y)
{
    double s, nu;
    int i;
    for (i = 0; i < dim; i++)
        if (!isfinite(x[i])) return ORC_ROW_NONFINITE;
    s = sum_sq(x, dim);
    if (s == 0.0) return ORC_ROW_ZERO_NORM;
    if (!isfinite(s)) return ORC_ROW_NONFINITE;
    nu = sqrt(s);
    for (i = 0; i < dim; i++) y[i] = oracle_bf16_round(x[i] / nu);
    /* a row can round to all zeros only if every x_i/nu < 2^-134; treat as zero norm */
    if (sum_sq(y, dim) == 0.0) return ORC_ROW_ZERO_NORM;
    return ORC_ROW_OK;
}

static double l2norm(const double *y, int dim)
{
    double s = 0.0;
    int i;
    for (i = 0; i < dim; i++) s = s + y[i] * y[i];
    return sqrt(s);
}

/* Convert one input row to fp64: fp32 (is_bf16 = 0) or raw bf16 bit patterns (is_bf16 = 1). */
static void load_row(const void *src, int is_bf16, int64_t row, int dim, double *out)
{
    int i;
    if (is_bf16) {
        const uint16_t *p = (const uint16_t *)src + row * (int64_t)dim;
        for (i = 0; i < dim; i++) {
            uint32_t u = ((uint32_t)p[i]) << 16;
            float f;
            memcpy(&f, &u, 4);
            out[i] = (double)f;
        }
    } else {
        const float *p = (const float *)src + row * (int64_t)dim;
        for (i = 0; i < dim; i++) out[i] = (double)p[i];
    }
}

oracle_cache *oracle_create(int dim, int64_t entry_capacity, int64_t latent_capacity,
                            int64_t latent_bytes, int num_k, const int *k_values,
                            const double *thresholds, int k_bias)
{
    oracle_cache *c;
    int j;
    if (dim <= 0 || entry_capacity <= 0 || latent_capacity < 0 || latent_bytes < 0 ||
        num_k <= 0 || num_k > ORC_MAX_K || k_bias < 0)
        return NULL;
    for (j = 1; j < num_k; j++)
        if (k_values[j] <= k_values[j - 1] || thresholds[j] < thresholds[j - 1]) return NULL;
    if (k_values[0] <= 0) return NULL;
    c = (oracle_cache *)calloc(1, sizeof(*c));
    if (!c) return NULL;
    c->dim = dim;
    c->entry_capacity = entry_capacity;
    c->latent_capacity = latent_capacity;
    c->latent_bytes = latent_bytes;
    c->num_k = num_k;
    for (j = 0; j < num_k; j++) {
        c->k_values[j] = k_values[j];
        c->thresholds[j] = thresholds[j];
    }
    c->k_bias = k_bias;
    return c;
}

static void free_entry_payload(oracle_cache *c, oentry *e)
{
    int j;
    for (j = 0; j < c->num_k; j++) {
        free(e->lat[j]);
        e->lat[j] = NULL;
    }
    free(e->x);
    e->x = NULL;
}

void oracle_destroy(oracle_cache *c)
{
    int64_t i;
    if (!c) return;
    for (i = 0; i < c->n_e; i++) free_entry_payload(c, &c->e[i]);
    free(c->e);
    free(c);
}

/* LCBFU insertion: all present K of each valid row are stored, f = 0.
 * latents: n x num_k x latent_bytes bytes or NULL (entries stored without payload bytes).
 * present: n bitmasks (bit j = k_values[j] present) or NULL (all K).
 * If the valid rows do not fit (entries or items), returns ORC_E_FULL with no state change. */
int oracle_insert(oracle_cache *c, int64_t n, const void *emb, int emb_is_bf16,
                  const unsigned char *latents, const uint8_t *present,
                  uint64_t *out_ids, int32_t *row_status)
{
    int64_t r, n_valid = 0, n_items = 0;
    double *x, *y;
    int *st;
    unsigned full_mask = (1u << c->num_k) - 1u;
    if (n < 0 || (n > 0 && !emb)) return ORC_E_INVALID_ARG;
    x = (double *)malloc(sizeof(double) * c->dim);
    y = (double *)malloc(sizeof(double) * c->dim * (n > 0 ? n : 1));
    st = (int *)malloc(sizeof(int) * (n > 0 ? n : 1));
    if (!x || !y || !st) {
        free(x); free(y); free(st);
        return ORC_E_OOM;
    }
    for (r = 0; r < n; r++) {
        unsigned m = present ? (present[r] & full_mask) : full_mask;
        load_row(emb, emb_is_bf16, r, c->dim, x);
        st[r] = normalise_row(x, c->dim, y + r * c->dim);
        if (st[r] == ORC_ROW_OK && m == 0) st[r] = ORC_ROW_NO_ITEMS;
        if (st[r] == ORC_ROW_OK) {
            int j;
            n_valid++;
            for (j = 0; j < c->num_k; j++) n_items += (m >> j) & 1u;
        }
    }
    if (c->live_entries + n_valid > c->entry_capacity ||
        c->live_items + n_items > c->latent_capacity) {
        free(x); free(y); free(st);
        return ORC_E_FULL;
    }
    if (c->n_e + n_valid > c->cap_e) {
        int64_t nc = c->cap_e ? c->cap_e : 64;
        oentry *ne;
        while (nc < c->n_e + n_valid) nc *= 2;
        ne = (oentry *)realloc(c->e, sizeof(oentry) * nc);
        if (!ne) {
            free(x); free(y); free(st);
            return ORC_E_OOM;
        }
        c->e = ne;
        c->cap_e = nc;
    }
    for (r = 0; r < n; r++) {
        oentry *e;
        unsigned m;
        int j;
        if (row_status) row_status[r] = st[r];
        if (st[r] != ORC_ROW_OK) {
            if (out_ids) out_ids[r] = ORC_NO_ID;
            continue;
        }
        m = present ? (present[r] & full_mask) : full_mask;
        e = &c->e[c->n_e++];
        memset(e, 0, sizeof(*e));
        e->id = c->next_id++;
        e->live = 1;
        e->x = (double *)malloc(sizeof(double) * c->dim);
        memcpy(e->x, y + r * c->dim, sizeof(double) * c->dim);
        e->nrm = l2norm(e->x, c->dim);
        for (j = 0; j < c->num_k; j++) {
            e->present[j] = (m >> j) & 1u;
            e->f[j] = 0;
            e->last[j] = c->clock;
            e->lat[j] = NULL;
            if (e->present[j] && latents && c->latent_bytes > 0) {
                e->lat[j] = (unsigned char *)malloc((size_t)c->latent_bytes);
                memcpy(e->lat[j], latents + ((size_t)r * c->num_k + j) * c->latent_bytes,
                       (size_t)c->latent_bytes);
            }
            if (e->present[j]) c->live_items++;
        }
        c->live_entries++;
        if (out_ids) out_ids[r] = e->id;
    }
    free(x); free(y); free(st);
    return ORC_OK;
}

/* Cosine similarity of a normalised query (q, nq) with entry e, all fp64. */
static double cosine(const oracle_cache *c, const double *q, double nq, const oentry *e)
{
    double d = 0.0;
    int i;
    for (i = 0; i < c->dim; i++) d = d + q[i] * e->x[i];
    return d / (nq * e->nrm);
}

typedef struct {
    double s;
    uint64_t id;
    int64_t idx;
} scored;

/* total order (s desc, id asc) -- reading R3 */
static int cmp_scored(const void *a, const void *b)
{
    const scored *x = (const scored *)a, *y = (const scored *)b;
    if (x->s > y->s) return -1;
    if (x->s < y->s) return 1;
    if (x->id < y->id) return -1;
    if (x->id > y->id) return 1;
    return 0;
}

/* Fig. 11 cache_selector with the table in c and the knob k_bias (R20).
 * Returns the bucket index j* (-1 = miss, K = 0). */
static int select_bucket(const oracle_cache *c, double s)
{
    double cl = s;
    int j, jstar = -1;
    if (cl > 1.0) cl = 1.0;
    if (cl < -1.0) cl = -1.0;
    for (j = 0; j < c->num_k; j++)
        if (cl > c->thresholds[j]) jstar = j;   /* largest j with s > thr[j] (strict) */
    if (jstar >= 0) {
        jstar += c->k_bias;
        if (jstar > c->num_k - 1) jstar = c->num_k - 1;
    }
    return jstar;
}

int oracle_select_k(const oracle_cache *c, double s)
{
    int j = select_bucket(c, s);
    return j < 0 ? 0 : c->k_values[j];
}

/* Hole rule: the present K with the largest value <= K*; -1 if none (reading R7). */
static int resolve_bucket(const oracle_cache *c, const oentry *e, int jstar)
{
    int j, best = -1;
    if (jstar < 0) return -1;
    for (j = 0; j < c->num_k; j++)
        if (e->present[j] && c->k_values[j] <= c->k_values[jstar]) best = j;
    return best;
}

/* Alg. 1 lines 4-8 for a batch of b queries.
 *   out_ids[b*topk], out_scores[b*topk] : top-k by (s desc, id asc); s reported clamped to
 *                                         [-1,1] (R4); none -> ORC_NO_ID / -inf
 *   out_raw[b*topk]                     : unclamped fp64 scores (may be NULL)
 *   out_k[b]                            : K actually used (after the hole rule), 0 = miss
 *   out_kstar[b]                        : K* from the threshold map before holes (may be NULL)
 *   latent_out[b*latent_bytes]          : row i written iff out_k[i] > 0 and bytes stored
 *   apply_counters                      : 1 -> f[e1][K_used] += 1 after the batch (R8, R9)
 */
int oracle_query(oracle_cache *c, int64_t b, const void *queries, int q_is_bf16, int topk,
                 uint64_t *out_ids, double *out_scores, double *out_raw, int32_t *out_k,
                 int32_t *out_kstar, unsigned char *latent_out, int32_t *row_status,
                 int apply_counters)
{
    double *x, *q;
    scored *all;
    int64_t i, r, n_live = 0;
    int64_t *hit_idx;
    int *hit_j;
    int any_bad = 0;
    if (b < 0 || topk <= 0 || (b > 0 && !queries)) return ORC_E_INVALID_ARG;
    x = (double *)malloc(sizeof(double) * c->dim);
    q = (double *)malloc(sizeof(double) * c->dim);
    all = (scored *)malloc(sizeof(scored) * (c->n_e > 0 ? c->n_e : 1));
    hit_idx = (int64_t *)malloc(sizeof(int64_t) * (b > 0 ? b : 1));
    hit_j = (int *)malloc(sizeof(int) * (b > 0 ? b : 1));
    if (!x || !q || !all || !hit_idx || !hit_j) {
        free(x); free(q); free(all); free(hit_idx); free(hit_j);
        return ORC_E_OOM;
    }
    for (r = 0; r < b; r++) {
        int st, t, jstar, jused;
        double nq;
        load_row(queries, q_is_bf16, r, c->dim, x);
        st = normalise_row(x, c->dim, q);
        if (row_status) row_status[r] = st;
        hit_idx[r] = -1;
        hit_j[r] = -1;
        for (t = 0; t < topk; t++) {
            out_ids[r * topk + t] = ORC_NO_ID;
            out_scores[r * topk + t] = -INFINITY;
            if (out_raw) out_raw[r * topk + t] = -INFINITY;
        }
        out_k[r] = 0;
        if (out_kstar) out_kstar[r] = 0;
        if (st != ORC_ROW_OK) {
            any_bad = 1;
            continue;
        }
        nq = l2norm(q, c->dim);
        n_live = 0;
        for (i = 0; i < c->n_e; i++) {
            if (!c->e[i].live) continue;
            all[n_live].s = cosine(c, q, nq, &c->e[i]);
            all[n_live].id = c->e[i].id;
            all[n_live].idx = i;
            n_live++;
        }
        qsort(all, (size_t)n_live, sizeof(scored), cmp_scored);
        for (t = 0; t < topk && t < n_live; t++) {
            double s = all[t].s;
            out_ids[r * topk + t] = all[t].id;
            if (out_raw) out_raw[r * topk + t] = s;
            out_scores[r * topk + t] = s > 1.0 ? 1.0 : (s < -1.0 ? -1.0 : s);
        }
        if (n_live == 0) continue;   /* empty cache: miss */
        jstar = select_bucket(c, all[0].s);
        if (out_kstar) out_kstar[r] = jstar < 0 ? 0 : c->k_values[jstar];
        jused = resolve_bucket(c, &c->e[all[0].idx], jstar);
        if (jused < 0) continue;     /* miss or every K <= K* is a hole */
        out_k[r] = c->k_values[jused];
        hit_idx[r] = all[0].idx;
        hit_j[r] = jused;
        if (latent_out && c->e[all[0].idx].lat[jused])
            memcpy(latent_out + (size_t)r * c->latent_bytes, c->e[all[0].idx].lat[jused],
                   (size_t)c->latent_bytes);
    }
    if (apply_counters) {
        c->clock++;   /* one query batch = one tick of the LRU clock */
        for (r = 0; r < b; r++)
            if (hit_idx[r] >= 0) {
                c->e[hit_idx[r]].f[hit_j[r]] += 1;
                c->e[hit_idx[r]].last[hit_j[r]] = c->clock;
            }
    }
    free(x); free(q); free(all); free(hit_idx); free(hit_j);
    return any_bad ? ORC_E_BAD_ROWS : ORC_OK;
}

static oentry *find_id(oracle_cache *c, uint64_t id)
{
    int64_t i;
    for (i = 0; i < c->n_e; i++)
        if (c->e[i].id == id) return c->e[i].live ? &c->e[i] : NULL;
    return NULL;
}

/* Record the accesses of one query batch chosen elsewhere (the parity harness adopts an
 * accepted GPU choice for queries whose top-1 is within tolerance, so multi-round counter
 * state stays comparable).  Like a query with apply_counters, it ticks the LRU clock once. */
int oracle_record_access(oracle_cache *c, int64_t n, const uint64_t *ids, const int32_t *ks)
{
    int64_t r;
    c->clock++;
    for (r = 0; r < n; r++) {
        oentry *e;
        int j, jj = -1;
        if (ks[r] == 0) continue;
        e = find_id(c, ids[r]);
        if (!e) return ORC_E_INVALID_ARG;
        for (j = 0; j < c->num_k; j++)
            if (c->k_values[j] == ks[r]) jj = j;
        if (jj < 0 || !e->present[jj]) return ORC_E_INVALID_ARG;
        e->f[jj] += 1;
        e->last[jj] = c->clock;
    }
    return ORC_OK;
}

/* Test hook: set the access count f of item (id, K_j) (e.g. past the GPU key's saturation
 * point, reading R11, which no test could reach through queries). */
int oracle_set_count(oracle_cache *c, uint64_t id, int32_t j, uint64_t f)
{
    oentry *e = find_id(c, id);
    if (!e || j < 0 || j >= c->num_k || !e->present[j]) return ORC_E_INVALID_ARG;
    e->f[j] = f;
    return ORC_OK;
}

/* Advance the LRU clock by one batch without accesses (a query batch with no hits). */
void oracle_tick(oracle_cache *c) { c->clock++; }

/* fp64 cosine of the (normalised, bf16-rounded) query row with a given live entry id. */
double oracle_score_id(oracle_cache *c, const void *query, int q_is_bf16, uint64_t id)
{
    double *x, *q, s;
    oentry *e = find_id(c, id);
    if (!e) return NAN;
    x = (double *)malloc(sizeof(double) * c->dim);
    q = (double *)malloc(sizeof(double) * c->dim);
    load_row(query, q_is_bf16, 0, c->dim, x);
    if (normalise_row(x, c->dim, q) != ORC_ROW_OK) {
        free(x); free(q);
        return NAN;
    }
    s = cosine(c, q, l2norm(q, c->dim), e);
    free(x); free(q);
    return s;
}

typedef struct {
    uint64_t score;   /* f_i x K_i */
    uint64_t id;
    int j;
    int64_t idx;
} item;

/* eviction order: (f x K, id, K) ascending -- reading R11 */
static int cmp_item(const void *a, const void *b)
{
    const item *x = (const item *)a, *y = (const item *)b;
    if (x->score != y->score) return x->score < y->score ? -1 : 1;
    if (x->id != y->id) return x->id < y->id ? -1 : 1;
    return x->j < y->j ? -1 : (x->j > y->j ? 1 : 0);
}

/* Policy scores (ascending = evicted first; ties by (id, K), reading R11 / SPEC S:341):
 *   0 LCBFU  f_i x K_i
 *   1 LRU    clock of the last access (insert clock if never accessed)
 *   2 LFU    f_i
 *   3 FIFO   0 -- the id (insertion sequence) decides */
static uint64_t policy_score(const oracle_cache *c, const oentry *e, int j, int policy)
{
    switch (policy) {
    case 1: return e->last[j];
    case 2: return e->f[j];
    case 3: return 0;
    default: return e->f[j] * (uint64_t)c->k_values[j];
    }
}

int oracle_evict_policy(oracle_cache *c, int64_t n, int policy, uint64_t *out_evicted,
                        uint64_t *out_dirty_ids, int64_t *out_n_dirty);

/* LCBFU eviction of the n lowest-scored items, then dirty-prompt removal.
 *   out_evicted[n]  : (id << 3 | j) in eviction order (ascending key); may be NULL
 *   out_dirty_ids   : ids of removed entries, ascending; capacity n (a dirty entry needs at
 *                     least one evicted item); may be NULL
 *   out_n_dirty     : number of entries removed */
int oracle_evict(oracle_cache *c, int64_t n, uint64_t *out_evicted, uint64_t *out_dirty_ids,
                 int64_t *out_n_dirty)
{
    return oracle_evict_policy(c, n, 0, out_evicted, out_dirty_ids, out_n_dirty);
}

/* Eviction of the n items with the smallest policy score (see policy_score). */
int oracle_evict_policy(oracle_cache *c, int64_t n, int policy, uint64_t *out_evicted,
                        uint64_t *out_dirty_ids, int64_t *out_n_dirty)
{
    item *it;
    int64_t i, m = 0, nd = 0;
    if (n < 0 || policy < 0 || policy > 3) return ORC_E_INVALID_ARG;
    if (n > c->live_items) return ORC_E_EVICT_RANGE;
    it = (item *)malloc(sizeof(item) * (c->live_items > 0 ? c->live_items : 1));
    if (!it) return ORC_E_OOM;
    for (i = 0; i < c->n_e; i++) {
        int j;
        if (!c->e[i].live) continue;
        for (j = 0; j < c->num_k; j++) {
            if (!c->e[i].present[j]) continue;
            it[m].score = policy_score(c, &c->e[i], j, policy);
            it[m].id = c->e[i].id;
            it[m].j = j;
            it[m].idx = i;
            m++;
        }
    }
    qsort(it, (size_t)m, sizeof(item), cmp_item);
    for (i = 0; i < n; i++) {
        oentry *e = &c->e[it[i].idx];
        e->present[it[i].j] = 0;
        free(e->lat[it[i].j]);
        e->lat[it[i].j] = NULL;
        c->live_items--;
        if (out_evicted) out_evicted[i] = (it[i].id << 3) | (uint64_t)it[i].j;
    }
    /* dirty: every K of the prompt is a hole -> remove from the index */
    for (i = 0; i < c->n_e; i++) {
        int j, any = 0;
        oentry *e = &c->e[i];
        if (!e->live) continue;
        for (j = 0; j < c->num_k; j++) any |= e->present[j];
        if (!any) {
            e->live = 0;
            free_entry_payload(c, e);
            c->live_entries--;
            if (out_dirty_ids) out_dirty_ids[nd] = e->id;
            nd++;
        }
    }
    if (out_n_dirty) *out_n_dirty = nd;
    free(it);
    return ORC_OK;
}

/* Entry-granularity eviction (SURVEY 8(b) evict_granularity = entry, reading c10 / DESIGN R24):
 * the score of a live entry is its items' policy scores aggregated over its PRESENT K --
 *   0 LCBFU  sum_j f_j x K_j   (the "segmented reduction" of the north_star)
 *   1 LRU    max_j last_j      (an entry is as recent as its most recently used state)
 *   2 LFU    sum_j f_j
 *   3 FIFO   0                 (the id decides)
 * Entries are ordered by (score, id) ascending and the first n are removed whole: every
 * stored state freed, the prompt gone from the index.
 *   out_ids[n] : removed entry ids in eviction order; may be NULL
 * n > live entries -> ORC_E_EVICT_RANGE. */
typedef struct {
    uint64_t score;
    uint64_t id;
    int64_t idx;
} entry_rank;

static int cmp_entry(const void *a, const void *b)
{
    const entry_rank *x = (const entry_rank *)a, *y = (const entry_rank *)b;
    if (x->score != y->score) return x->score < y->score ? -1 : 1;
    return x->id < y->id ? -1 : (x->id > y->id ? 1 : 0);
}

int oracle_evict_entries(oracle_cache *c, int64_t n, int policy, uint64_t *out_ids)
{
    entry_rank *er;
    int64_t i, m = 0;
    if (n < 0 || policy < 0 || policy > 3) return ORC_E_INVALID_ARG;
    if (n > c->live_entries) return ORC_E_EVICT_RANGE;
    er = (entry_rank *)malloc(sizeof(entry_rank) * (c->live_entries > 0 ? c->live_entries : 1));
    if (!er) return ORC_E_OOM;
    for (i = 0; i < c->n_e; i++) {
        int j;
        uint64_t sc = 0;
        const oentry *e = &c->e[i];
        if (!e->live) continue;
        for (j = 0; j < c->num_k; j++) {
            uint64_t v;
            if (!e->present[j]) continue;
            v = policy_score(c, e, j, policy);
            if (policy == 1) sc = v > sc ? v : sc;
            else sc += v;
        }
        er[m].score = sc;
        er[m].id = e->id;
        er[m].idx = i;
        m++;
    }
    qsort(er, (size_t)m, sizeof(entry_rank), cmp_entry);
    for (i = 0; i < n; i++) {
        int j;
        oentry *e = &c->e[er[i].idx];
        for (j = 0; j < c->num_k; j++) {
            if (!e->present[j]) continue;
            e->present[j] = 0;
            c->live_items--;
        }
        e->live = 0;
        free_entry_payload(c, e);
        c->live_entries--;
        if (out_ids) out_ids[i] = er[i].id;
    }
    free(er);
    return ORC_OK;
}

/* ---- inspection helpers for tests ---- */
int64_t oracle_live_entries(const oracle_cache *c) { return c->live_entries; }
int64_t oracle_live_items(const oracle_cache *c) { return c->live_items; }
uint64_t oracle_next_id(const oracle_cache *c) { return c->next_id; }

/* stored fp64 row of entry id; returns 0 on success */
int oracle_get_row(oracle_cache *c, uint64_t id, double *out)
{
    oentry *e = find_id(c, id);
    if (!e) return ORC_E_INVALID_ARG;
    memcpy(out, e->x, sizeof(double) * c->dim);
    return ORC_OK;
}

/* counters f[num_k] and presence mask of entry id */
int oracle_get_meta(oracle_cache *c, uint64_t id, uint64_t *f, uint32_t *present_mask)
{
    int j;
    uint32_t m = 0;
    oentry *e = find_id(c, id);
    if (!e) return ORC_E_INVALID_ARG;
    for (j = 0; j < c->num_k; j++) {
        if (f) f[j] = e->f[j];
        m |= (uint32_t)(e->present[j] ? 1u : 0u) << j;
    }
    if (present_mask) *present_mask = m;
    return ORC_OK;
}

uint64_t oracle_clock(const oracle_cache *c) { return c->clock; }

/* last-access clocks of entry id (num_k values) */
int oracle_get_last(oracle_cache *c, uint64_t id, uint64_t *last)
{
    int j;
    oentry *e = find_id(c, id);
    if (!e) return ORC_E_INVALID_ARG;
    for (j = 0; j < c->num_k; j++) last[j] = e->last[j];
    return ORC_OK;
}

/* plain fp64 normalise + bf16 round of one row (exposed so tests can pin it directly) */
int oracle_normalise(int dim, const double *x, double *y) { return normalise_row(x, dim, y); }
