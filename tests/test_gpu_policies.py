"""GPU parity of the eviction policies (LCBFU and its FIFO / LRU / LFU baselines, SURVEY
NEXT-2): the same radix-select kernels with policy keys, against the oracle, over several
query / evict / insert rounds (integer keys: exact, including eviction order)."""
import numpy as np
import pytest
import torch

import synth
from tests.parity import check_batch, gpu_to_numpy

pytestmark = pytest.mark.gpu
L = 128


@pytest.mark.parametrize("policy", [0, 1, 2, 3])
def test_policy_rounds_parity(oracle_mod, policy):
    from paper_2312_04429_b200 import binding as B
    n = 500
    emb, cl = synth.entries(n, seed=60 + policy)
    pres = synth.present_masks(n, seed=60, hole_frac=0.2)
    lat = synth.latents_np(np.arange(n), 5, L, seed=60)
    g = B.NirvanaCache(entry_capacity=n + 200, latent_capacity=5 * n + 1000, dim=768, latent_bytes=L)
    g.set_evict_policy(policy)
    o = oracle_mod.OracleCache(dim=768, entry_capacity=n + 200, latent_capacity=5 * n + 1000, latent_bytes=L)
    g.insert(torch.from_numpy(emb).cuda(), torch.from_numpy(lat).cuda(), present=pres)
    o.insert(emb, latents=lat, present=pres)
    rng = np.random.default_rng(policy)
    extra_row = 0
    for rnd in range(5):
        for _ in range(2):
            q, _, _ = synth.queries(emb, cl, 150, seed=1000 * policy + rnd * 10 + _)
            out = gpu_to_numpy(g.query(torch.from_numpy(q).cuda(), topk=1))
            check_batch(out, o, q, 1, expected_latent=None)
        nev = int(rng.integers(50, 400))
        ev, d = g.evict(nev)
        rc, oev, od = o.evict(nev, policy=policy)
        assert rc == 0 and np.array_equal(ev, oev) and np.array_equal(d, od), (policy, rnd)
        # re-insert fresh prompts so LRU sees items with later insert clocks
        m = 20
        ne, _ = synth.entries(m, seed=900 + rnd)
        nl = synth.latents_np(np.arange(m) + 10_000 + extra_row, 5, L, seed=61)
        extra_row += m
        gi, _ = g.insert(torch.from_numpy(ne).cuda(), torch.from_numpy(nl).cuda())
        rc, oi, _ = o.insert(ne, latents=nl)
        assert np.array_equal(gi, oi)


@pytest.mark.parametrize("policy", [1, 2])
def test_policy_sharded_equals_single(policy):
    """LRU clocks and LFU counts are updated over the peer path by the requesting rank:
    virtual shards must evict exactly what one cache evicts."""
    from paper_2312_04429_b200 import binding as B, sharded as S
    n = 800
    emb, cl = synth.entries(n, seed=70)
    single = B.NirvanaCache(entry_capacity=n, dim=768, latent_bytes=L)
    vs = S.VirtualShards(3, entry_capacity=n, dim=768, latent_bytes=L)
    single.set_evict_policy(policy)
    vs.set_evict_policy(policy)
    et = torch.from_numpy(emb).cuda()
    single.insert(et)
    vs.insert(et)
    for r in range(3):
        q, _, _ = synth.queries(emb, cl, 96, seed=71 + r)
        qt = torch.from_numpy(q).cuda()
        single.query(qt, latents=False)
        vs.query(qt, latents=False)
        torch.cuda.synchronize()
    e1, d1 = single.evict(1234)
    e2, d2 = vs.evict(1234)
    assert np.array_equal(e1, e2) and np.array_equal(d1, d2)   # global eviction order


@pytest.mark.parametrize("policy", [0, 1, 2, 3])
def test_entry_granularity_rounds_parity(oracle_mod, policy):
    """Entry granularity (R24): whole entries by the aggregated policy score, same radix
    select with one key per entry; evicted ids, order and the survivors' results exact."""
    from paper_2312_04429_b200 import binding as B
    n = 600
    emb, cl = synth.entries(n, seed=80 + policy)
    pres = synth.present_masks(n, seed=80, hole_frac=0.3)
    lat = synth.latents_np(np.arange(n), 5, L, seed=80)
    g = B.NirvanaCache(entry_capacity=n + 200, latent_capacity=5 * n + 1000, dim=768, latent_bytes=L,
                       evict_granularity=B.EVICT_ENTRY)
    g.set_evict_policy(policy)
    o = oracle_mod.OracleCache(dim=768, entry_capacity=n + 200, latent_capacity=5 * n + 1000, latent_bytes=L)
    g.insert(torch.from_numpy(emb).cuda(), torch.from_numpy(lat).cuda(), present=pres)
    o.insert(emb, latents=lat, present=pres)
    rng = np.random.default_rng(10 + policy)
    mask_of = {i: int(pres[i]) for i in range(n)}
    lat_of = {i: lat[i] for i in range(n)}
    for rnd in range(4):
        for i in range(2):
            q, _, _ = synth.queries(emb, cl, 160, seed=2000 * policy + rnd * 10 + i)
            out = gpu_to_numpy(g.query(torch.from_numpy(q).cuda(), topk=1))
            check_batch(out, o, q, 1, expected_latent=lambda id_, K: lat_of[id_][synth.K_VALUES.index(K)])
        nev = int(rng.integers(20, 120))
        items_before = g.live_items
        ev, dirty = g.evict(nev)
        rc, oev = o.evict_entries(nev, policy=policy)
        assert rc == 0 and np.array_equal(ev, oev), (policy, rnd)
        assert np.array_equal(dirty, np.sort(oev))
        assert g.live_entries == o.live_entries and g.live_items == o.live_items
        assert items_before - g.live_items == sum(bin(mask_of[int(i)]).count("1") for i in ev)
        m = 30
        ne, _ = synth.entries(m, seed=950 + rnd)
        nl = synth.latents_np(np.arange(m) + 20_000 + 100 * rnd, 5, L, seed=81)
        gi, _ = g.insert(torch.from_numpy(ne).cuda(), torch.from_numpy(nl).cuda())
        rc, oi, _ = o.insert(ne, latents=nl)
        assert np.array_equal(gi, oi)
        for r, id_ in enumerate(gi):
            mask_of[int(id_)], lat_of[int(id_)] = 31, nl[r]
    with pytest.raises(B.CacheError):
        g.evict(g.live_entries + 1)


@pytest.mark.parametrize("policy", [0, 1])
def test_entry_granularity_sharded_equals_single(policy):
    from paper_2312_04429_b200 import binding as B, sharded as S
    n = 900
    emb, cl = synth.entries(n, seed=90)
    single = B.NirvanaCache(entry_capacity=n, dim=768, latent_bytes=L, evict_granularity=B.EVICT_ENTRY)
    vs = S.VirtualShards(4, entry_capacity=n, dim=768, latent_bytes=L, evict_granularity=B.EVICT_ENTRY)
    single.set_evict_policy(policy)
    vs.set_evict_policy(policy)
    et = torch.from_numpy(emb).cuda()
    single.insert(et)
    vs.insert(et)
    for r in range(3):
        q, _, _ = synth.queries(emb, cl, 128, seed=91 + r)
        qt = torch.from_numpy(q).cuda()
        single.query(qt, latents=False)
        vs.query(qt, latents=False)
        torch.cuda.synchronize()
    e1, d1 = single.evict(333)
    e2, d2 = vs.evict(333)
    assert np.array_equal(e1, e2) and np.array_equal(d1, d2)   # global eviction order
    assert vs.stats()["live_entries"] == single.live_entries == n - 333
