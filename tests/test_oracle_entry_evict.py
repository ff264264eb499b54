"""Pins of the oracle's entry-granularity eviction (SURVEY 8(b) evict_granularity, reading c10 /
DESIGN R24): n whole entries with the smallest aggregated policy score -- LCBFU sum f*K (the
segmented reduction), LRU max last access, LFU sum f, FIFO 0 -- ties by id."""
import numpy as np
import pytest

import synth


def _cache(oracle_mod, n=8, dim=16):
    return oracle_mod.OracleCache(dim=dim, entry_capacity=n)


def test_entry_score_is_the_sum_not_the_min(oracle_mod):
    """id0 holds K=5 (f=0) and K=25 (f=100): items 0 and 2500, entry score 2500 (P:602-603's
    100 x 25 example).  id1 holds K=10 only with f=50: 500.  Item granularity evicts id0's
    K=5 item first (score 0); entry granularity removes id1 first (500 < 2500)."""
    H = synth.hand_vectors(16)
    o = _cache(oracle_mod)
    o.insert(H[[1, 2]], present=np.array([(1 << 0) | (1 << 4), 1 << 1], np.uint8))
    o.record_access(np.zeros(100, np.uint64), np.full(100, 25, np.int32))
    o.record_access(np.ones(50, np.uint64), np.full(50, 10, np.int32))
    rc, ids = o.evict_entries(1, policy=oracle_mod.LCBFU)
    assert rc == 0 and list(ids) == [1]
    assert o.live_entries == 1 and o.live_items == 2
    o2 = _cache(oracle_mod)
    o2.insert(H[[1, 2]], present=np.array([(1 << 0) | (1 << 4), 1 << 1], np.uint8))
    o2.record_access(np.zeros(100, np.uint64), np.full(100, 25, np.int32))
    o2.record_access(np.ones(50, np.uint64), np.full(50, 10, np.int32))
    rc, ev, dirty = o2.evict(1, policy=oracle_mod.LCBFU)
    assert rc == 0 and list(ev) == [(0 << 3) | 0] and len(dirty) == 0


def test_lru_entry_is_as_recent_as_its_newest_state(oracle_mod):
    """LRU aggregates by max: id0 touched at clock 1 (K=5) and never again; id1 inserted at
    clock 0, its K=10 state touched at clock 2 -> id0 (max 1) goes before id1 (max 2)."""
    H = synth.hand_vectors(16)
    o = _cache(oracle_mod)
    o.insert(H[[1, 2]])                                                      # clock 0
    o.record_access(np.array([0], np.uint64), np.array([5], np.int32))      # clock 1
    o.record_access(np.array([1], np.uint64), np.array([10], np.int32))     # clock 2
    assert list(o.last(0)) == [1, 0, 0, 0, 0] and list(o.last(1)) == [0, 2, 0, 0, 0]
    rc, ids = o.evict_entries(1, policy=oracle_mod.LRU)
    assert rc == 0 and list(ids) == [0]


def test_fifo_entries_in_insertion_order(oracle_mod):
    H = synth.hand_vectors(16)
    o = _cache(oracle_mod)
    o.insert(H[[1, 2, 3, 4]])
    o.record_access(np.zeros(9, np.uint64), np.full(9, 25, np.int32))
    rc, ids = o.evict_entries(3, policy=oracle_mod.FIFO)
    assert rc == 0 and list(ids) == [0, 1, 2] and o.live_entries == 1 and o.live_items == 5


@pytest.mark.parametrize("policy", [0, 1, 2, 3])
def test_single_state_entries_reduce_to_item_eviction(oracle_mod, policy):
    """Special case: every entry stores exactly one K -> the entry score equals its only
    item's score and the (score, id) order equals the item order (score, id, K), so entry
    eviction of n = item eviction of n (whose victims are then all dirty)."""
    n = 60
    emb, _ = synth.entries(n, seed=7, dim=16)
    rng = np.random.default_rng(policy)
    pres = (1 << rng.integers(0, 5, n)).astype(np.uint8)
    kv = np.array(synth.K_VALUES)
    seq = [rng.integers(0, n, 30).astype(np.uint64) for _ in range(4)]
    res = []
    for mode in ("item", "entry"):
        o = _cache(oracle_mod, n=n)
        o.insert(emb, present=pres)
        for ids in seq:
            ks = kv[np.log2(pres[ids.astype(np.int64)]).astype(int)].astype(np.int32)
            o.record_access(ids, ks)
        if mode == "item":
            rc, ev, dirty = o.evict(17, policy=policy)
            assert rc == 0 and np.array_equal(np.sort(ev >> np.uint64(3)), dirty)
            res.append(ev >> np.uint64(3))
        else:
            rc, ids = o.evict_entries(17, policy=policy)
            assert rc == 0
            res.append(ids)
    assert np.array_equal(res[0], res[1])


@pytest.mark.parametrize("policy", [0, 1, 2, 3])
def test_entry_eviction_optimal_by_brute_force(oracle_mod, policy):
    """max(evicted keys) < min(surviving keys), keys recomputed here from the per-item
    counters / clocks the oracle reports (get_meta, last) -- not from its eviction code."""
    n = 50
    emb, _ = synth.entries(n, seed=11, dim=16)
    rng = np.random.default_rng(100 + policy)
    pres = synth.present_masks(n, seed=11, hole_frac=0.5)
    o = _cache(oracle_mod, n=n)
    o.insert(emb, present=pres)
    kv = np.array(synth.K_VALUES)
    for _ in range(6):
        ids = rng.integers(0, n, 25)
        ks = []
        for i in ids:
            js = [j for j in range(5) if (pres[i] >> j) & 1]
            ks.append(kv[rng.choice(js)])
        o.record_access(ids.astype(np.uint64), np.array(ks, np.int32))

    def key(i):
        f, m = o.meta(i)
        last = o.last(i)
        items = [j for j in range(5) if (m >> j) & 1]
        if policy == 0:
            s = sum(int(f[j]) * int(kv[j]) for j in items)
        elif policy == 1:
            s = max(int(last[j]) for j in items)
        elif policy == 2:
            s = sum(int(f[j]) for j in items)
        else:
            s = 0
        return (s, i)

    keys = {i: key(i) for i in range(n)}
    items_before = o.live_items
    rc, ev = o.evict_entries(19, policy=policy)
    assert rc == 0 and len(ev) == 19
    assert [keys[int(i)] for i in ev] == sorted(keys[int(i)] for i in ev)        # eviction order
    survivors = set(range(n)) - {int(i) for i in ev}
    assert max(keys[int(i)] for i in ev) < min(keys[i] for i in survivors)
    assert o.live_entries == n - 19
    assert items_before - o.live_items == sum(bin(int(pres[int(i)])).count("1") for i in ev)
    q = emb[[int(i) for i in ev]]
    res = o.query(q, topk=1, want_latents=False, apply_counters=False)
    assert not set(int(x) for x in res["ids"][:, 0]) & {int(i) for i in ev}   # gone from the index


def test_entry_eviction_range(oracle_mod):
    H = synth.hand_vectors(16)
    o = _cache(oracle_mod)
    o.insert(H[[1, 2]])
    assert o.evict_entries(3)[0] == 4                     # ORC_E_EVICT_RANGE: n > live entries
    assert o.live_entries == 2
    rc, ids = o.evict_entries(0)
    assert rc == 0 and len(ids) == 0 and o.live_entries == 2
