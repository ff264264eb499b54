/*
 * nirvana_cache_debug.h -- test-only entry points of libnirvana_cache.so (not the product
 * API).  They expose intermediate results of the lookup so each kernel can be checked on its
 * own against a plain reference.
 */
#ifndef NIRVANA_CACHE_DEBUG_H
#define NIRVANA_CACHE_DEBUG_H

#include "nirvana_cache.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Dense scan values of the tensor-core main loop: out[i*ld + e] = fl(<q~_i, x~_e> *
 * inv_norm(x~_e)) for every query i < b and entry slot e < entry_hwm (the value the fused
 * top-k epilogue ranks; NaN for empty slots).  queries: device pointer b x dim (q_dtype);
 * out: device pointer, b x ld floats, ld >= round_up(entry_hwm, 256).  Asynchronous.
 * Returns CACHE_E_UNSUPPORTED when the tcgen05 kernel is unavailable. */
cache_status cache_debug_tc_scores(cache_t *c, int64_t b, const void *queries, int32_t q_dtype,
                                   float *out, int64_t ld, void *stream);

/* Slot of entry `id` (host-synchronous), -1 if not live. */
int64_t cache_debug_slot_of(cache_t *c, uint64_t id);

/* The eviction path's GPU sort on its own: sorts n u64 keys (device pointer) ascending in
 * place (LSD radix, 8 x 8-bit stable passes).  Synchronises `stream`. */
cache_status cache_debug_sort_u64(uint64_t *keys, int64_t n, void *stream);
/* The same with the options the eviction uses: keys in [base, base + 2^bits) sorted by
 * ceil(bits/8) LSD passes over key - base (small = 0: 3 launches per pass; small = 2: the
 * one-launch cooperative version), or (small = 1, n <= 16384) the one-CTA bitonic sort in
 * shared memory.  Synchronises `stream`. */
cache_status cache_debug_sort_u64_ex(uint64_t *keys, int64_t n, int32_t bits, uint64_t base, int32_t small,
                                     void *stream);
/* Statistics of the last cache_evict (fused select + apply): out4 = {levels, full sweeps of
 * the slot columns, level at which candidates were compacted (0 = none), candidates}. */
cache_status cache_debug_evict_stats(cache_t *c, int64_t *out4);
/* Cap the fused eviction's candidate buffer (cap < 0: automatic), so the tests can force the
 * paths that compact late or never. */
cache_status cache_debug_set_evict_cand_cap(cache_t *c, int64_t cap);
/* The single-sweep window of cache_evict (a systematic 1/S sample estimates the n-th key, the
 * level-0 sweep compacts every key below the estimate, the selection finishes on them): with
 * set != 0, stride -1 = automatic, 0 = off (the two-sweep path), S = a fixed 1/S sample (S = 1:
 * the whole cache, an exact estimate; a huge S: a biased estimate, so the tests reach the
 * fall-back).  *last (may be null) = the last eviction's window: 0 off, 1 used, 2 missed. */
cache_status cache_debug_evict_window(cache_t *c, int32_t stride, int32_t set, int32_t *last);
/* Set the LCBFU access count f of item (id, K_j) (host-synchronous): the tests reach counts no
 * query stream could (the key saturation of reading R11). */
cache_status cache_debug_set_count(cache_t *c, uint64_t id, int32_t j, uint32_t f);

#ifdef __cplusplus
}
#endif
#endif
