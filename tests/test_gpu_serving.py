"""NEXT-1 on the GPU: the serving loop driving the CUDA library against the oracle's own
loop (oracle/serving.py) request by request -- every request's entry and K are validated by
the parity harness against the fp64 oracle (which adopts the accepted decision on near-ties),
then both loops account and admit independently: per-request K and latency, per-step evicted
and dirty ids and admitted prompts, and the totals must be identical."""
import numpy as np
import pytest

import synth
from paper_2312_04429_b200.serving import GpuCache, LatencyParams, ServingLoop
from tests.parity import check_batch, gpu_to_numpy

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("entries,items,b,policy", [(300, 1200, 64, 0), (300, 1200, 64, 1), (50, 200, 128, 0)])
def test_gpu_serving_per_request_parity(oracle_mod, entries, items, b, policy):
    from oracle.serving import OracleServing
    from paper_2312_04429_b200 import binding as B
    universe, cl = synth.entries(3000, seed=77)
    g = B.NirvanaCache(entry_capacity=entries, latent_capacity=items, dim=768, latent_bytes=0)
    g.set_evict_policy(policy)
    gc = GpuCache(g)
    prod = ServingLoop(gc, synth.K_VALUES, LatencyParams(), keep_log=True)
    orc = oracle_mod.OracleCache(dim=768, entry_capacity=entries, latent_capacity=items)
    ref = OracleServing(orc, synth.K_VALUES, entry_capacity=entries, item_capacity=items, policy=policy)
    hits = 0
    for i in range(15):
        q, _, _ = synth.queries(universe, cl, b, seed=300 + i)
        prod.step(q)
        out = gpu_to_numpy(gc.last_out)
        rep = check_batch(out, orc, q, 1, expected_latent=None)   # every request vs the oracle
        hits += rep["hits"]
        ref.step(q, out["k"])
        a, e = prod.log[-1], ref.log[-1]
        assert np.array_equal(a["k"], e["k"]) and a["latency"] == e["latency"], i
        assert np.array_equal(a["evicted"], e["evicted"]), (i, a["evicted"][:8], e["evicted"][:8])
        assert np.array_equal(a["dirty"], e["dirty"]) and a["admitted"] == e["admitted"], i
        assert g.live_items == orc.live_items and g.live_entries == orc.live_entries, i
    s = prod.report.summary(prod.lat)
    assert {k: prod.report.hits_at.get(k, 0) for k in synth.K_VALUES} == ref.served_at
    assert s["f_c"] == pytest.approx(ref.f_c(), abs=1e-12) and prod.report.latencies == ref.latencies
    assert hits > 0 and s["evicted_items"] > 0


def test_peek_counts_no_access(oracle_mod):
    """cache_query_peek reports what cache_query_batch would (ids, scores, K) and leaves the
    counters, the LRU clock and hence every later eviction untouched."""
    import torch
    from paper_2312_04429_b200 import binding as B
    emb, cl = synth.entries(2000, seed=31)
    a = B.NirvanaCache(entry_capacity=2000, latent_capacity=10_000, dim=768, latent_bytes=0)
    c = B.NirvanaCache(entry_capacity=2000, latent_capacity=10_000, dim=768, latent_bytes=0)
    for x in (a, c):
        x.set_evict_policy(1)   # LRU: sensitive to clock ticks as well as counters
        x.insert(torch.from_numpy(emb).cuda())
    q = torch.from_numpy(synth.queries(emb, cl, 512, seed=32)[0]).cuda()
    p = a.peek(q)
    r = c.query(q, latents=False)
    assert torch.equal(p["ids"], r["ids"]) and torch.equal(p["k"], r["k"]) and torch.equal(p["scores"], r["scores"])
    q2 = torch.from_numpy(synth.queries(emb, cl, 256, seed=33)[0]).cuda()
    a.query(q2, latents=False)
    a.peek(q)                       # more peeks: nothing changes
    c2 = B.NirvanaCache(entry_capacity=2000, latent_capacity=10_000, dim=768, latent_bytes=0)
    c2.set_evict_policy(1)
    c2.insert(torch.from_numpy(emb).cuda())
    c2.query(q2, latents=False)     # the same history without the peeks
    assert np.array_equal(a.evict(3000)[0], c2.evict(3000)[0])
    assert a.stats()["queries"] == c2.stats()["queries"]


def test_serving_with_match_predictor():
    """Alg. 1 with the predictor: predicted misses cost exactly C and take
    no search; the predictor is retrained on > 5% change; its precision c_p and
    the wasted-search fraction are reported."""
    from paper_2312_04429_b200 import binding as B
    universe, cl = synth.entries(20_000, seed=5)
    g = B.NirvanaCache(entry_capacity=2000, latent_capacity=10_000, dim=768, latent_bytes=0)
    loop = ServingLoop(GpuCache(g), synth.K_VALUES, LatencyParams(), use_predictor=True)
    for i in range(20):
        q, _, _ = synth.queries(universe, cl, 128, seed=700 + i)
        loop.step(q)
    ps = loop.predictor_summary()
    s = loop.report.summary(loop.lat)
    assert ps["retrains"] >= 2 and ps["predicted_true"] + ps["predicted_false"] <= s["requests"]
    assert 0.0 <= ps["precision_c_p"] <= 1.0 and s["f_c"] == pytest.approx(s["f_c_from_steps"], abs=1e-12)
    n_scratch_pred = sum(1 for x in loop.report.latencies if x == loop.lat.C)
    assert n_scratch_pred >= ps["predicted_false"]


def test_policy_direction_lcbfu_first():
    """SPEC acceptance #6 / Table 3(b) direction: on a skewed-similarity stream at
    two capacities LCBFU saves at least as much compute as LFU and FIFO, and >= LRU - 0.01."""
    from paper_2312_04429_b200 import binding as B
    universe, cl = synth.entries(50_000, seed=2024)
    streams = [synth.queries(universe, cl, 256, seed=9000 + i)[0] for i in range(60)]
    for cap in (2000, 8000):
        fc = {}
        for policy in (0, 1, 2, 3):
            g = B.NirvanaCache(entry_capacity=cap, latent_capacity=5 * cap, dim=768, latent_bytes=0)
            g.set_evict_policy(policy)
            loop = ServingLoop(GpuCache(g), synth.K_VALUES, LatencyParams())
            for q in streams:
                loop.step(q)
            fc[policy] = loop.report.f_c(50)
        assert fc[0] >= fc[2] - 1e-12 and fc[0] >= fc[3] - 1e-12 and fc[0] >= fc[1] - 0.01, (cap, fc)
