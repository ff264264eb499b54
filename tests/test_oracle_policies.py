"""Pins of the oracle's comparison eviction policies: FIFO / LRU / LFU
 next to LCBFU."""
import numpy as np

import synth


def _cache(oracle_mod, n=4, k_values=synth.K_VALUES, thresholds=(0.65, 0.75, 0.85, 0.90, 0.95)):
    return oracle_mod.OracleCache(dim=16, entry_capacity=n, k_values=k_values, thresholds=thresholds[:len(k_values)])


def test_lfu_ignores_k_and_lcbfu_does_not(oracle_mod):
    """LFU picks f=1 before f=2 regardless of K; LCBFU weighs by K."""
    H = synth.hand_vectors(16)
    for policy, want in ((oracle_mod.LFU, (0 << 3) | 4), (oracle_mod.LCBFU, (1 << 3) | 0)):
        o = _cache(oracle_mod)
        o.insert(H[[0, 2]], present=np.array([1 << 4, 1 << 0], np.uint8))   # id0: K=25 only; id1: K=5 only
        o.record_access(np.array([0], np.uint64), np.array([25], np.int32))                 # f=1 at K=25
        o.record_access(np.array([1, 1], np.uint64), np.array([5, 5], np.int32))            # f=2 at K=5
        rc, ev, _ = o.evict(1, policy=policy)
        # LFU: (f=1,id0,K25) < (f=2,id1,K5); LCBFU: 1*25=25 > 2*5=10 -> the K=5 item goes
        assert rc == 0 and list(ev) == [want], policy


def test_fifo_evicts_by_insertion_sequence(oracle_mod):
    """FIFO picks insert_seq = 0 first, whatever the counters say."""
    H = synth.hand_vectors(16)
    o = _cache(oracle_mod)
    o.insert(H[[1, 2, 3]])
    o.record_access(np.array([0, 0, 0], np.uint64), np.array([25, 25, 25], np.int32))
    rc, ev, dirty = o.evict(7, policy=oracle_mod.FIFO)
    assert list(ev) == [(0 << 3) | j for j in range(5)] + [(1 << 3) | 0, (1 << 3) | 1]
    assert list(dirty) == [0]


def test_lru_uses_batch_clock_and_insert_time(oracle_mod):
    """LRU evicts the least recently accessed item; never-accessed items carry their insert
    clock, so an old hot item can outlive a fresh cold one only if it was touched later."""
    H = synth.hand_vectors(16)
    o = _cache(oracle_mod)
    o.insert(H[[1]], present=np.array([1], np.uint8))               # id0 (K=5), clock 0
    o.record_access(np.array([0], np.uint64), np.array([5], np.int32))   # clock 1: id0 touched
    o.tick()                                                        # clock 2: batch with no hits
    o.insert(H[[2]], present=np.array([1], np.uint8))               # id1 inserted at clock 2
    assert list(o.last(0))[0] == 1 and list(o.last(1))[0] == 2
    rc, ev, _ = o.evict(1, policy=oracle_mod.LRU)
    assert list(ev) == [0]                                          # last access 1 < 2


def test_degenerate_policy_equivalence(oracle_mod):
    """with all K equal and all f equal, LCBFU's victims have the same scores as LFU's
    (single-K table; identical tie-break -> identical victim sets)."""
    emb, _ = synth.entries(40, seed=3, dim=16)
    res = []
    for policy in (oracle_mod.LCBFU, oracle_mod.LFU):
        o = _cache(oracle_mod, n=40, k_values=(10,), thresholds=(0.5,))
        o.insert(emb)
        o.record_access(np.arange(40, dtype=np.uint64), np.full(40, 10, np.int32))
        res.append(o.evict(13, policy=policy)[1])
    assert np.array_equal(res[0], res[1])


def test_policy_optimality_fuzz(oracle_mod):
    """Every policy: evicted keys <= every surviving key (exhaustive scan)."""
    rng = np.random.default_rng(8)
    emb, _ = synth.entries(50, seed=8, dim=16)
    for policy in (oracle_mod.LRU, oracle_mod.LFU, oracle_mod.FIFO):
        o = _cache(oracle_mod, n=50)
        o.insert(emb, present=synth.present_masks(50, seed=policy, hole_frac=0.3))
        live = list(range(50))
        for _ in range(60):
            e = int(rng.choice(live))
            _, m = o.meta(e)
            j = int(rng.choice([j for j in range(5) if m >> j & 1]))
            o.record_access(np.array([e], np.uint64), np.array([synth.K_VALUES[j]], np.int32))
        keys = {}
        for e in live:
            f, m = o.meta(e)
            last = o.last(e)
            for j in range(5):
                if m >> j & 1:
                    s = {oracle_mod.LRU: int(last[j]), oracle_mod.LFU: int(f[j]), oracle_mod.FIFO: 0}[policy]
                    keys[(e, j)] = (s, e, j)
        rc, ev, _ = o.evict(37, policy=policy)
        gone = {(int(x) >> 3, int(x) & 7) for x in ev}
        assert max(keys[g] for g in gone) < min(v for k, v in keys.items() if k not in gone)
