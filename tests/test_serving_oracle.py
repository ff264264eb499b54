"""NEXT-1 oracle loop (oracle/serving.py) pinned by a hand-worked case (P:297-304, P:317-324,
P:602-611), and the product's ServingLoop host logic compared with it step by step on CPU (the
fp64 oracle plays the cache on both sides: per-request K and latency, evicted and dirty ids,
admitted prompts, f_C), including batches larger than the whole cache."""
import numpy as np
import pytest

import synth
from paper_2312_04429_b200.serving import LatencyParams, ServingLoop
from tests.test_serving import OracleAdapter

KV = synth.K_VALUES


def _unit(i, dim=64):
    v = np.zeros((1, dim), np.float32)
    v[0, i] = 1.0
    return v


def test_oracle_serving_hand_case(oracle_mod):
    from oracle.serving import OracleServing
    orc = oracle_mod.OracleCache(dim=64, entry_capacity=2, latent_capacity=10)
    loop = OracleServing(orc, KV, entry_capacity=2, item_capacity=10)

    def step(q):
        r = orc.query(q, topk=1, want_latents=False, apply_counters=True)   # Alg. 1 lookup
        loop.step(q, r["k"])
        return loop.log[-1]

    s = step(np.vstack([_unit(0), _unit(1)]))            # cold cache: two misses, both admitted
    assert list(s["k"]) == [0, 0] and s["admitted"] == 2 and len(s["evicted"]) == 0
    s = step(_unit(0))                                    # exact repeat: s = 1 > 0.95 -> K = 25
    assert list(s["k"]) == [25] and s["latency"] == [0.1 + 8.59 * 25 / 50 + 0.05]
    # a new orthogonal prompt (s = 0): miss.  Storage full -> evict |K| = 5 items first: the
    # lowest f*K keys (f*K, id, j): id 0 j 0..3 (f 0), id 1 j 0 (f 0); id 0's K=25 item has
    # f*K = 25.  No entry empties, so no entry slot frees and the prompt is not admitted.
    s = step(_unit(2))
    assert list(s["k"]) == [0] and s["latency"] == [0.1 + 8.59]
    assert list(s["evicted"]) == [0, 1, 2, 3, 8] and len(s["dirty"]) == 0 and s["admitted"] == 0
    # again: entries short by one -> 5 more items: id 1 j 1..4 (f 0), then id 0 j 4 (f*K = 25);
    # both entries are now dirty and the prompt is admitted
    s = step(_unit(2))
    assert list(s["evicted"]) == [9, 10, 11, 12, 4] and list(s["dirty"]) == [0, 1] and s["admitted"] == 1
    assert orc.live_entries == 1 and orc.live_items == 5
    # accounting: 5 requests, one served at K = 25 -> h_opt(25) = 0.2, f_C = 0.2 * 25 / 50
    assert loop.requests == 5 and loop.served_at[25] == 1
    assert loop.hit_rate() == pytest.approx(0.2) and loop.f_c() == pytest.approx(0.1)


@pytest.mark.parametrize("entries,items,b,policy", [(60, 250, 32, 0), (60, 250, 32, 1), (8, 30, 40, 0),
                                                    (50, 120, 16, 3)])
def test_product_loop_matches_oracle_loop_per_step(oracle_mod, entries, items, b, policy):
    """Both loops driven by identical oracle caches: every step's per-request K and latency,
    evicted / dirty ids and admitted count are equal, and so are the totals.  (8, 30, 40): a
    batch of 40 misses against a 6-prompt cache -- the eviction is capped at the live items
    and the admission is partial (it used to raise EVICT_RANGE)."""
    from oracle.serving import OracleServing
    universe, cl = synth.entries(400, seed=11, dim=64)
    cache = OracleAdapter(oracle_mod, 64, entries=entries, items=items, policy=policy)
    prod = ServingLoop(cache, KV, LatencyParams(), keep_log=True)
    orc = oracle_mod.OracleCache(dim=64, entry_capacity=entries, latent_capacity=items)
    ref = OracleServing(orc, KV, entry_capacity=entries, item_capacity=items, policy=policy)
    for i in range(12):
        q, _, _ = synth.queries(universe, cl, b, seed=5 + i)
        prod.step(q)
        r = orc.query(q, topk=1, want_latents=False, apply_counters=True)
        ref.step(q, r["k"])
        a, e = prod.log[-1], ref.log[-1]
        assert np.array_equal(a["k"], e["k"]), i
        assert a["latency"] == e["latency"], i
        assert np.array_equal(a["evicted"], e["evicted"]) and np.array_equal(a["dirty"], e["dirty"]), i
        assert a["admitted"] == e["admitted"], i
    s = prod.report.summary(prod.lat)
    assert s["requests"] == ref.requests
    assert {k: prod.report.hits_at.get(k, 0) for k in KV} == ref.served_at
    assert s["f_c"] == pytest.approx(ref.f_c(), abs=1e-12) and s["hit_rate"] == pytest.approx(ref.hit_rate(), abs=1e-12)
    assert prod.report.latencies == ref.latencies
    assert cache.o.live_items == orc.live_items and cache.o.live_entries == orc.live_entries
