"""Query slicing of cache_query_batch (cache_set_query_slices): the scan as several launches
over query slices with the earlier slices' finalize + gather on a side stream.  A scheduling
choice only -- every output, counter and later eviction must be bit-identical to one launch
(R9: each query sees the pre-batch state), and the sliced path must match the oracle."""
import numpy as np
import pytest
import torch

import synth
from tests.parity import check_batch, gpu_to_numpy

pytestmark = pytest.mark.gpu

L = 256


@pytest.fixture(scope="module")
def B():
    from paper_2312_04429_b200 import binding
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return binding


def _cache(B, emb, lat, pres, slices):
    n = emb.shape[0]
    g = B.NirvanaCache(entry_capacity=n, dim=768, latent_bytes=L)
    g.insert(torch.from_numpy(emb).cuda(), torch.from_numpy(lat).cuda(), pres)
    g.set_query_slices(slices)
    return g


def _run(g, qs, topk):
    outs = []
    for q in qs:   # successive batches reuse the slice workspace and the side stream
        outs.append(gpu_to_numpy(g.query(torch.from_numpy(q).cuda(), topk=topk)))
    torch.cuda.synchronize()
    return outs


@pytest.mark.parametrize("topk", [1, 4])
@pytest.mark.parametrize("b", [1100, 4096])
def test_slices_bit_identical_to_one_launch(B, oracle_mod, b, topk):
    n = 20_000
    emb, cl = synth.entries(n, seed=611)
    pres = synth.present_masks(n, seed=611)
    lat = synth.latents_np(np.arange(n), 5, L, seed=611)
    qs = [synth.queries(emb, cl, b, seed=612 + r)[0] for r in range(2)]
    ref_g = _cache(B, emb, lat, pres, 1)
    ref = _run(ref_g, qs, topk)
    hit_ids = np.unique(np.concatenate([o["ids"][o["k"] > 0, 0] for o in ref]))
    def metas(g):
        return [(tuple(int(x) for x in f), m) for f, m in (g.meta(int(i)) for i in hit_ids)]
    ref_meta = metas(ref_g)
    ref_ev = ref_g.evict(300)
    # 0 = auto (one launch); b = 1,100 with 3 / 8 requested
    # gives slices of 512 + 512 + 76 (the last on the single-CTA kernel) / 4 x 256 + 76
    for slices in (0, 2, 3, 4, 8):
        g = _cache(B, emb, lat, pres, slices)
        outs = _run(g, qs, topk)
        for o, r in zip(outs, ref):
            for key in ("ids", "scores", "k", "status"):
                assert np.array_equal(o[key], r[key]), (slices, key)
            hit = r["k"] > 0   # rows with K = 0 are left untouched (uninitialised buffers)
            assert np.array_equal(o["latents"][hit], r["latents"][hit]), slices
        assert metas(g) == ref_meta, slices
        ev = g.evict(300)
        assert np.array_equal(ev[0], ref_ev[0]) and np.array_equal(ev[1], ref_ev[1]), slices
        g.close()
    # and the sliced path against the oracle on sampled rows of the first batch
    o = oracle_mod.OracleCache(dim=768, entry_capacity=n, latent_bytes=L)
    o.insert(emb, latents=lat, present=pres)
    g = _cache(B, emb, lat, pres, 2)
    out = gpu_to_numpy(g.query(torch.from_numpy(qs[0]).cuda(), topk=topk))
    rows = sorted(set(np.random.default_rng(b).choice(b, 24, replace=False).tolist()) | {0, b - 1, 767, 768})
    rep = check_batch(out, o, qs[0], topk, rows=rows, adopt=False,
                      expected_latent=lambda e, k: lat[e, synth.K_VALUES.index(k)])
    assert rep["max_dscore"] < 1e-4


def test_slices_argument_checks(B):
    g = B.NirvanaCache(entry_capacity=16, dim=768, latent_bytes=0)
    for bad in (-1, 9):
        with pytest.raises(B.CacheError):
            g.set_query_slices(bad)
    g.set_query_slices(8)
    g.set_query_slices(0)


def test_evict_without_lists_matches(B):
    """cache_evict with NULL output lists (counts only) leaves exactly the state the listed call
    does: same live counts, same later lookups, same next eviction (entry and item mode)."""
    from paper_2312_04429_b200.binding import _lib, _ptr
    n = 6000
    emb, cl = synth.entries(n, seed=631)
    pres = synth.present_masks(n, seed=631)
    lat = synth.latents_np(np.arange(n), 5, L, seed=631)
    q = synth.queries(emb, cl, 700, seed=632)[0]
    for gran in (0, 1):
        a, b = _cache(B, emb, lat, pres, 0), _cache(B, emb, lat, pres, 0)
        for g in (a, b):
            g.set_evict_granularity(gran)
            g.query(torch.from_numpy(q).cuda())
        k = 500 if gran else 4000
        a.evict(k)
        nd = np.zeros(1, dtype=np.int64)
        assert _lib.cache_evict(b._h, k, None, None, _ptr(nd), None) == 0
        assert a.stats() == b.stats()
        ra, rb = (gpu_to_numpy(g.query(torch.from_numpy(q).cuda())) for g in (a, b))
        for key in ("ids", "scores", "k"):
            assert np.array_equal(ra[key], rb[key]), (gran, key)
        hit = ra["k"] > 0
        assert np.array_equal(ra["latents"][hit], rb["latents"][hit])
        ea, eb = a.evict(k // 2), b.evict(k // 2)
        assert np.array_equal(ea[0], eb[0]) and np.array_equal(ea[1], eb[1])
        a.close()
        b.close()
