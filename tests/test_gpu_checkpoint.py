"""Checkpoint / resume (cache_save / cache_load; the paper's cache persists in EFS
files + a Qdrant collection): a handle restored from a snapshot answers every later
call exactly as the saved handle does -- lookups (ids, scores, K, latent bytes), LCBFU / LRU
counters, evictions (order and dirty lists), insertions (ids, slots) -- and the restored cache
still matches the fp64 oracle."""
import numpy as np
import pytest
import torch

import synth
from tests.parity import check_batch, gpu_to_numpy

pytestmark = pytest.mark.gpu
L = 64


def _same(a, b):
    for k in ("ids", "scores", "k"):
        assert torch.equal(a[k], b[k]), k
    if a.get("latents") is not None:   # gathered states of the hits (miss rows are not written)
        hit = a["k"] > 0
        assert torch.equal(a["latents"][hit], b["latents"][hit])


@pytest.mark.parametrize("policy,gran,alias", [(0, 0, False), (1, 0, False), (0, 1, False), (2, 0, True)])
def test_save_load_continues_identically(tmp_path, oracle_mod, policy, gran, alias):
    from paper_2312_04429_b200 import binding as B
    n = 1200
    emb, cl = synth.entries(n, seed=811)
    pres = synth.present_masks(n, seed=811, hole_frac=0.2)
    lat = synth.latents_np(np.arange(n), 5, L, seed=811)
    kw = dict(entry_capacity=n + 200, latent_capacity=(1024 if alias else 5 * (n + 200)), dim=768, latent_bytes=L,
              latent_alias=alias, evict_granularity=gran)
    g = B.NirvanaCache(**kw)
    g.set_evict_policy(policy)
    lat_t = None if alias else torch.from_numpy(lat).cuda()   # an aliased pool takes no insert payload
    g.insert(torch.from_numpy(emb).cuda(), lat_t, present=pres)
    for r in range(3):
        q, _, _ = synth.queries(emb, cl, 128, seed=820 + r)
        g.query(torch.from_numpy(q).cuda(), topk=4)
    g.evict(g.evict_units // 10)
    ne, _ = synth.entries(60, seed=830)
    g.insert(torch.from_numpy(ne).cuda(),
             None if alias else torch.from_numpy(synth.latents_np(np.arange(n, n + 60), 5, L, seed=811)).cuda())
    g.set_thresholds([0.6, 0.7, 0.8, 0.9, 0.97])
    g.train_predictor(epochs=5)
    path = str(tmp_path / "cache.snap")
    g.save(path)
    h = B.NirvanaCache.load(path)
    assert g.stats() == h.stats()
    assert h.granularity == gran and h.k_values == g.k_values and h.latent_capacity == g.latent_capacity
    for r in range(3):   # lookups, then maintenance, on both handles in lockstep
        q, _, _ = synth.queries(emb, cl, 96, seed=840 + r)
        qt = torch.from_numpy(q).cuda()
        _same(g.query(qt, topk=4), h.query(qt, topk=4))
        fg, mg = g.predict(qt)
        fh, mh = h.predict(qt)
        assert torch.equal(fg, fh) and torch.equal(mg, mh)
        nev = max(1, g.evict_units // 20)
        eg, dg = g.evict(nev)
        eh, dh = h.evict(nev)
        assert np.array_equal(eg, eh) and np.array_equal(dg, dh)
        ne, _ = synth.entries(len(dg), seed=850 + r)
        if len(ne):
            lt = None if alias else torch.from_numpy(synth.latents_np(np.arange(len(ne)), 5, L, seed=851 + r)).cuda()
            ig = g.insert(torch.from_numpy(ne).cuda(), lt)
            ih = h.insert(torch.from_numpy(ne).cuda(), lt)
            assert np.array_equal(np.asarray(ig[0] if isinstance(ig, tuple) else ig),
                                  np.asarray(ih[0] if isinstance(ih, tuple) else ih))
        assert g.stats() == h.stats()
    for id_ in range(0, n + 200, 37):   # per-(entry, K) counters and presence masks
        try:
            fa, ma = g.meta(id_)
        except B.CacheError:
            with pytest.raises(B.CacheError):
                h.meta(id_)
            continue
        fb, mb = h.meta(id_)
        assert np.array_equal(fa, fb) and ma == mb


def test_restored_cache_matches_oracle(tmp_path, oracle_mod):
    from paper_2312_04429_b200 import binding as B
    n = 1000
    emb, cl = synth.entries(n, seed=861)
    pres = synth.present_masks(n, seed=861)
    lat = synth.latents_np(np.arange(n), 5, L, seed=861)
    g = B.NirvanaCache(entry_capacity=n, dim=768, latent_bytes=L)
    g.insert(torch.from_numpy(emb).cuda(), torch.from_numpy(lat).cuda(), present=pres)
    o = oracle_mod.OracleCache(dim=768, entry_capacity=n, latent_bytes=L)
    o.insert(emb, latents=lat, present=pres)
    q0, _, _ = synth.queries(emb, cl, 64, seed=862)
    check_batch(gpu_to_numpy(g.query(torch.from_numpy(q0).cuda(), topk=1)), o, q0, 1,
                expected_latent=lambda e, k: lat[e, synth.K_VALUES.index(k)])
    path = str(tmp_path / "c.snap")
    g.save(path)
    del g
    h = B.NirvanaCache.load(path)
    q1, _, _ = synth.queries(emb, cl, 64, seed=863)
    check_batch(gpu_to_numpy(h.query(torch.from_numpy(q1).cuda(), topk=1)), o, q1, 1,
                expected_latent=lambda e, k: lat[e, synth.K_VALUES.index(k)])
    ev, dirty = h.evict(40)
    rc, oev, od = o.evict(40)
    assert rc == 0 and np.array_equal(ev, oev) and np.array_equal(dirty, od)


def test_save_without_latents_and_bad_files(tmp_path):
    from paper_2312_04429_b200 import binding as B
    n = 300
    emb, cl = synth.entries(n, seed=871)
    lat = synth.latents_np(np.arange(n), 5, L, seed=871)
    g = B.NirvanaCache(entry_capacity=n, dim=768, latent_bytes=L)
    g.insert(torch.from_numpy(emb).cuda(), torch.from_numpy(lat).cuda())
    full, slim = str(tmp_path / "full.snap"), str(tmp_path / "slim.snap")
    g.save(full)
    g.save(slim, with_latents=False)
    import os
    assert os.path.getsize(full) - os.path.getsize(slim) >= 5 * n * L
    h = B.NirvanaCache.load(slim)
    q = torch.from_numpy(emb[:32]).cuda()
    a, b = g.query(q), h.query(q)
    assert torch.equal(a["ids"], b["ids"]) and torch.equal(a["k"], b["k"])   # latents not restored
    data = open(full, "rb").read()
    trunc = str(tmp_path / "trunc.snap")
    open(trunc, "wb").write(data[: len(data) // 2])
    for bad in (trunc, str(tmp_path / "missing.snap")):
        with pytest.raises(B.CacheError) as ei:
            B.NirvanaCache.load(bad)
        assert ei.value.code == B.E_INVALID_ARG
