"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on seeded inputs."""
import numpy as np
import pytest
import torch

import synth
from tests.parity import check_batch, check_stored_row, gpu_to_numpy

pytestmark = pytest.mark.gpu

L_SMALL = 256


@pytest.fixture(scope="module")
def B():
    from paper_2312_04429_b200 import binding
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return binding


def _bf16_bits(x: np.ndarray) -> np.ndarray:
    return (x.astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)


def _make(B, oracle_mod, n, dim=768, L=L_SMALL, seed=1, present=None, cap=None, lcap=None, k_bias=0):
    emb, cl = synth.entries(n, seed=seed, dim=dim)
    lat = synth.latents_np(np.arange(n), 5, L, seed=seed) if L else None
    g = B.NirvanaCache(entry_capacity=cap or max(n, 1), latent_capacity=lcap, dim=dim, latent_bytes=L,
                       k_bias=k_bias)
    o = oracle_mod.OracleCache(dim=dim, entry_capacity=cap or max(n, 1), latent_capacity=lcap,
                               latent_bytes=L, k_bias=k_bias)
    if n:
        gid, gst = g.insert(torch.from_numpy(emb).cuda(), torch.from_numpy(lat).cuda() if L else None, present)
        rc, oid, ost = o.insert(emb, latents=lat, present=present)
        assert rc == 0 and np.array_equal(gid, oid) and np.array_equal(gst, ost)
    return g, o, emb, cl, lat


SCORERS = ["stream", "tc", "tc1"]   # CUDA-core scan; tcgen05 (CTA pairs above 128 queries); single-CTA tcgen05


def _set(g, B, scorer):
    g.set_scorer({"stream": B.SCORER_STREAM, "tc": B.SCORER_TC, "tc1": B.SCORER_TC_SINGLE}[scorer])


def test_stored_rows_bit_identical(B, oracle_mod):
    """Stored rows equal the oracle's plain index-order normalisation bit for bit, up to the
    proved summation-order accept set (tests/parity.py check_stored_row; expected count 0)."""
    g, o, emb, _, _ = _make(B, oracle_mod, 300, L=0, seed=3)
    accepted = sum(check_stored_row(g.row_bf16(i), emb[i], o.row(i)) for i in range(300))
    print(f"stored-row accept-set components: {accepted}")
    assert accepted == 0


@pytest.mark.parametrize("scorer", SCORERS)
def test_hand_cache_exact(B, oracle_mod, scorer):
    """Hand-worked exact cache H (tests/golden/hand_cache_H.txt): bit-exact scores and K."""
    H = synth.hand_vectors(768)
    g = B.NirvanaCache(entry_capacity=8, dim=768, latent_bytes=L_SMALL)
    _set(g, B, scorer)
    g.insert(torch.from_numpy(H[1:]).cuda())
    out = gpu_to_numpy(g.query(torch.from_numpy(H[[0, 2]]).cuda(), topk=4, latents=False))
    assert list(out["ids"][0]) == [3, 2, 0, 1] and list(out["scores"][0]) == [0.9375, 0.875, 0.75, 0.5]
    assert out["k"][0] == 20 and out["ids"][1, 0] == 1 and out["scores"][1, 0] == 1.0 and out["k"][1] == 25
    g1 = B.NirvanaCache(entry_capacity=8, dim=768, latent_bytes=L_SMALL)
    _set(g1, B, scorer)
    g1.insert(torch.from_numpy(H[1:2]).cuda())
    o1 = gpu_to_numpy(g1.query(torch.from_numpy(H[:1]).cuda(), topk=1, latents=False))
    assert o1["scores"][0, 0] == 0.75 and o1["k"][0] == 5          # strict boundary
    g.insert(torch.from_numpy(H[[0, 4]]).cuda())                    # u0 (id 4), dup u4 (id 5)
    o2 = gpu_to_numpy(g.query(torch.from_numpy(H[[0, 4]]).cuda(), topk=2, latents=False))
    assert o2["ids"][0, 0] == 4 and o2["k"][0] == 25
    assert list(o2["ids"][1]) == [3, 5] and o2["scores"][1, 0] == o2["scores"][1, 1] == 1.0
    for mask, want in ((0b00111, 15), (0b10000, 0)):               # holes, no fallback
        gh = B.NirvanaCache(entry_capacity=8, dim=768, latent_bytes=L_SMALL)
        _set(gh, B, scorer)
        gh.insert(torch.from_numpy(H[3:5]).cuda(), present=np.array([0b11111, mask], np.uint8))
        r = gpu_to_numpy(gh.query(torch.from_numpy(H[:1]).cuda(), topk=1, latents=False))
        assert r["ids"][0, 0] == 1 and r["k"][0] == want


@pytest.mark.parametrize("scorer", SCORERS)
@pytest.mark.parametrize("topk", [1, 5, 16])
def test_c1_parity(B, oracle_mod, scorer, topk):
    """C1: 1,000 entries x 768, 64 queries, latents, holes; two rounds with counters."""
    n = 1000
    pres = synth.present_masks(n, seed=5)
    g, o, emb, cl, lat = _make(B, oracle_mod, n, seed=5, present=pres)
    _set(g, B, scorer)
    q, _, _ = synth.queries(emb, cl, 64, seed=6)
    exp = lambda e, k: lat[e, synth.K_VALUES.index(k)]
    for rnd in range(2):
        out = gpu_to_numpy(g.query(torch.from_numpy(q).cuda(), topk=topk))
        rep = check_batch(out, o, q, topk, expected_latent=exp)
        assert rep["max_dscore"] < 1e-4, rep
        assert rep["hits"] > 20
    for e in range(n):
        gf, gm = g.meta(e)
        of, om = o.meta(e)
        assert gm == om and np.array_equal(gf, of), e


@pytest.mark.parametrize("scorer", SCORERS)
@pytest.mark.parametrize("n,b", [(1, 1), (255, 3), (257, 129), (300, 130), (777, 7), (1025, 257)])
def test_ragged_sizes(B, oracle_mod, scorer, n, b):
    g, o, emb, cl, lat = _make(B, oracle_mod, n, seed=n + b)
    _set(g, B, scorer)
    q, _, _ = synth.queries(emb, cl, b, seed=b)
    out = gpu_to_numpy(g.query(torch.from_numpy(q).cuda(), topk=min(4, 16)))
    check_batch(out, o, q, 4, expected_latent=lambda e, k: lat[e, synth.K_VALUES.index(k)])


@pytest.mark.parametrize("scorer", SCORERS)
@pytest.mark.parametrize("dim", [64, 128, 512, 1024])
def test_other_dims(B, oracle_mod, scorer, dim):
    """The whole path at other embedding widths (multiples of 64 up to the 1,024 maximum):
    stored rows bit-identical, ids / K / bytes within the contract, several tiles + a tail."""
    n, b = 700, 300
    g, o, emb, cl, lat = _make(B, oracle_mod, n, dim=dim, seed=dim)
    _set(g, B, scorer)
    for i in (0, 123, n - 1):
        assert check_stored_row(g.row_bf16(i), emb[i], o.row(i)) == 0
    q, _, _ = synth.queries(emb, cl, b, seed=dim + 1)
    out = gpu_to_numpy(g.query(torch.from_numpy(q).cuda(), topk=4))
    check_batch(out, o, q, 4, expected_latent=lambda e, k: lat[e, synth.K_VALUES.index(k)])


@pytest.mark.parametrize("scorer", SCORERS)
def test_edge_cases(B, oracle_mod, scorer):
    g = B.NirvanaCache(entry_capacity=16, dim=768, latent_bytes=L_SMALL)
    _set(g, B, scorer)
    q = torch.randn(5, 768, device="cuda")
    out = gpu_to_numpy(g.query(q, topk=3))                          # empty cache: all misses
    assert (out["ids"] == np.uint64(0xFFFFFFFFFFFFFFFF)).all() and (out["k"] == 0).all()
    assert np.isneginf(out["scores"]).all()
    emb, _ = synth.entries(2, seed=1)
    g.insert(torch.from_numpy(emb).cuda())
    q[1] = 0.0
    q[2, 5] = float("nan")
    out = gpu_to_numpy(g.query(q, topk=3))
    assert list(out["status"]) == [0, 2, 1, 0, 0]
    assert out["k"][1] == 0 and out["k"][2] == 0 and out["ids"][1, 0] == np.uint64(0xFFFFFFFFFFFFFFFF)
    assert out["ids"][0, 2] == np.uint64(0xFFFFFFFFFFFFFFFF)       # fewer live entries than topk
    bad = torch.from_numpy(emb).cuda().clone()
    bad[0] = 0.0
    ids, st = g.insert(bad)
    assert list(st) == [2, 0] and ids[0] == np.uint64(0xFFFFFFFFFFFFFFFF)


def test_full_and_errors(B):
    g = B.NirvanaCache(entry_capacity=4, latent_capacity=12, dim=768, latent_bytes=L_SMALL)
    emb, _ = synth.entries(6, seed=2)
    g.insert(torch.from_numpy(emb[:2]).cuda())
    with pytest.raises(B.CacheError) as e:
        g.insert(torch.from_numpy(emb[:3]).cuda())
    assert e.value.code == B.E_FULL and g.stats()["live_entries"] == 2
    with pytest.raises(B.CacheError) as e:
        g.evict(11)
    assert e.value.code == B.E_EVICT_RANGE
    with pytest.raises(B.CacheError) as e:
        g.query(torch.randn(2, 768, device="cuda"), topk=17)
    assert e.value.code == B.E_INVALID_ARG


@pytest.mark.parametrize("scorer", SCORERS)
def test_eviction_rounds_parity(B, oracle_mod, scorer):
    """Query rounds (counters) + LCBFU evictions + inserts: evicted sets, dirty lists, counters
    and subsequent lookups all equal the oracle's (integer keys: exact)."""
    n = 600
    pres = synth.present_masks(n, seed=9, hole_frac=0.2)
    g, o, emb, cl, lat = _make(B, oracle_mod, n, seed=9, present=pres, cap=700, lcap=3200)
    _set(g, B, scorer)
    rng = np.random.default_rng(9)
    for rnd in range(4):
        q, _, _ = synth.queries(emb, cl, 200, seed=100 + rnd)
        out = gpu_to_numpy(g.query(torch.from_numpy(q).cuda(), topk=1))
        live = lambda e: _live(o, e)
        check_batch(out, o, q, 1, expected_latent=lambda e, k: lat[e, synth.K_VALUES.index(k)])
        nev = int(rng.integers(1, 400))
        gev, gd = g.evict(nev)
        rc, oev, od = o.evict(nev)
        assert rc == 0 and np.array_equal(gev, oev) and np.array_equal(gd, od)
        st = g.stats()
        assert st["live_items"] == o.live_items and st["live_entries"] == o.live_entries
    # the whole-cache 2-hop path: evict everything
    n_all = o.live_items
    gev, gd = g.evict(n_all)
    rc, oev, od = o.evict(n_all)
    assert np.array_equal(gev, oev) and np.array_equal(gd, od) and g.stats()["live_entries"] == 0
    out = gpu_to_numpy(g.query(torch.from_numpy(emb[:4]).cuda(), topk=1))
    assert (out["k"] == 0).all()
    # slots are reused deterministically after eviction
    e2, c2 = synth.entries(50, seed=77)
    l2 = synth.latents_np(np.arange(50) + 10_000, 5, L_SMALL, seed=77)
    gid, _ = g.insert(torch.from_numpy(e2).cuda(), torch.from_numpy(l2).cuda())
    _, oid, _ = o.insert(e2, latents=l2)
    assert np.array_equal(gid, oid)
    q, _, _ = synth.queries(e2, c2, 40, seed=78)
    out = gpu_to_numpy(g.query(torch.from_numpy(q).cuda(), topk=2))
    check_batch(out, o, q, 2, expected_latent=lambda e, k: l2[e - int(gid[0]), synth.K_VALUES.index(k)])


def _live(o, e):
    try:
        o.meta(e)
        return True
    except KeyError:
        return False


def test_lcbfu_paper_example_on_gpu(B):
    """(K=25, f=100) scores 2500 > (K=5, f=200) = 1000 -> the K=5 item is evicted first."""
    H = synth.hand_vectors(768)
    g = B.NirvanaCache(entry_capacity=4, dim=768, latent_bytes=L_SMALL)
    g.insert(torch.from_numpy(H[[0, 2]]).cuda(), present=np.array([1 << 4, 1 << 0], np.uint8))
    qa = torch.from_numpy(np.repeat(H[:1], 100, 0)).cuda()       # u0 -> entry 0 at K=25
    qb = torch.from_numpy(np.repeat(H[2:3], 200, 0)).cuda()      # u2 -> entry 1 at K=5
    assert (g.query(qa)["k"] == 25).all().item() and (g.query(qb)["k"] == 5).all().item()
    assert list(g.meta(0)[0]) == [0, 0, 0, 0, 100] and list(g.meta(1)[0]) == [200, 0, 0, 0, 0]
    ev, dirty = g.evict(1)
    assert list(ev) == [(1 << 3) | 0] and list(dirty) == [1]


@pytest.mark.parametrize("scorer", SCORERS)
def test_host_variant_matches_device(B, oracle_mod, scorer):
    g, o, emb, cl, lat = _make(B, oracle_mod, 500, seed=12)
    _set(g, B, scorer)
    q, _, _ = synth.queries(emb, cl, 33, seed=13)
    d = gpu_to_numpy(g.query(torch.from_numpy(q).cuda(), topk=3))
    h = g.query_host(np.ascontiguousarray(q), topk=3)
    assert np.array_equal(d["ids"], h["ids"]) and np.array_equal(d["scores"], h["scores"])
    assert np.array_equal(d["k"], h["k"])
    for i in range(33):
        if d["k"][i] > 0:
            assert np.array_equal(d["latents"][i], h["latents"][i])


def test_scorers_agree_bitwise_on_ids(B, oracle_mod):
    """Stream and TC scorers: same entries and K wherever the oracle gap exceeds tau."""
    g, o, emb, cl, lat = _make(B, oracle_mod, 3000, seed=21, L=0)
    q, _, _ = synth.queries(emb, cl, 300, seed=22)
    qt = torch.from_numpy(q).cuda()
    g.set_scorer(B.SCORER_STREAM)
    a = gpu_to_numpy(g.query(qt, topk=1, latents=False))
    g.set_scorer(B.SCORER_TC)
    b = gpu_to_numpy(g.query(qt, topk=1, latents=False))
    assert np.mean(a["ids"][:, 0] == b["ids"][:, 0]) > 0.98
    assert np.max(np.abs(a["scores"] - b["scores"])) < 1e-4


def test_full_size_sampled_parity_c2(B, oracle_mod):
    """C2 at full size in the bench's launch configuration (100K entries, B = 4,096, TC path):
    (entry, K, score) of EVERY one of the 4,096 queries checked against the oracle's exact scan
    of all 100K entries (the host's threads, ~25 s), and the latent stamps of every hit."""
    n, b, L = 100_000, 4096, 32768
    emb, cl = synth.entries(n, seed=1001)
    pres = synth.present_masks(n, seed=1001)
    g = B.NirvanaCache(entry_capacity=n, dim=768, latent_bytes=L)
    for s in range(0, n, 8192):
        m = min(8192, n - s)
        lat = synth.latents_torch(s, m, 5, L, seed=1001, device="cuda")
        g.insert(torch.from_numpy(emb[s:s + m]).cuda(), lat, present=pres[s:s + m])
        del lat
    o = oracle_mod.OracleCache(dim=768, entry_capacity=n, latent_bytes=0)
    o.insert(emb, present=pres)
    q, _, _ = synth.queries(emb, cl, b, seed=1002)
    out = gpu_to_numpy(g.query(torch.from_numpy(q).cuda(), topk=1))
    hits = np.nonzero(out["k"] > 0)[0]
    assert 0.7 < len(hits) / b < 0.98
    for i in hits:                                                # stamp check on every hit row
        e, k = int(out["ids"][i, 0]), int(out["k"][i])
        exp = synth.latent_np([e], synth.K_VALUES.index(k), L, seed=1001)[0]
        assert np.array_equal(out["latents"][i], exp)
    rep = check_batch(out, o, q, 1, rows=list(range(b)), adopt=False)
    assert rep["checked"] == b
    print(rep)
    assert rep["max_dscore"] < 1e-4


def test_aliased_latent_pool(B, oracle_mod):
    """latent_alias = 1 (SURVEY 8(d) capacity decision for C4/C5): items read the declared
    slot CACHE_ALIAS_SLOT(id, j, cap) of a pre-filled pool; entries/K unaffected."""
    n, cap, L2 = 700, 37, 512
    emb, cl = synth.entries(n, seed=41)
    pres = synth.present_masks(n, seed=41, hole_frac=0.3)
    pool = synth.latents_np(np.arange(cap) + 90_000, 1, L2, seed=41)[:, 0]     # [cap][L]
    g = B.NirvanaCache(entry_capacity=n, latent_capacity=cap, dim=768, latent_bytes=L2, latent_alias=True)
    g.pool_write(0, torch.from_numpy(pool).cuda())
    g.insert(torch.from_numpy(emb).cuda(), None, present=pres)
    per_item = np.stack([np.stack([pool[B.alias_slot(e, j, cap)] for j in range(5)]) for e in range(n)])
    o = oracle_mod.OracleCache(dim=768, entry_capacity=n, latent_bytes=L2)
    o.insert(emb, latents=per_item, present=pres)
    q, _, _ = synth.queries(emb, cl, 130, seed=42)
    out = gpu_to_numpy(g.query(torch.from_numpy(q).cuda(), topk=2))
    check_batch(out, o, q, 2, expected_latent=lambda e, k: per_item[e, synth.K_VALUES.index(k)])
    ev, d = g.evict(900)
    rc, oev, od = o.evict(900)
    assert np.array_equal(ev, oev) and np.array_equal(d, od)
    with pytest.raises(B.CacheError):
        g.insert(torch.from_numpy(emb[:2]).cuda(), torch.zeros((2, 5, L2), dtype=torch.uint8, device="cuda"))


def test_full_size_sampled_parity_c3(B, oracle_mod):
    """C3's shape: 1M entries, B = 32 (the HBM-bound single-CTA scan, hundreds of partial lists
    per query to merge), top-4; all 32 queries, every rank, against the oracle's exact fp64 scan of
    all 1M entries, and the batch-wide properties for every query."""
    n, b = 1_000_000, 32
    emb, cl = synth.entries(n, seed=3001)
    g = B.NirvanaCache(entry_capacity=n, dim=768, latent_bytes=0, latent_capacity=5 * n)
    for s in range(0, n, 65536):
        g.insert(torch.from_numpy(emb[s:s + 65536]).cuda())
    q, _, _ = synth.queries(emb, cl, b, seed=3002)
    out = gpu_to_numpy(g.query(torch.from_numpy(q).cuda(), topk=4, latents=False))
    assert (np.diff(out["scores"], axis=1) <= 0).all()                 # best first
    assert (out["ids"] < n).all() and (out["status"] == 0).all()
    o = oracle_mod.OracleCache(dim=768, entry_capacity=n, latent_bytes=0)
    o.insert(emb)
    del emb
    rep = check_batch(out, o, q, 4, adopt=False)
    print(rep)
    assert rep["max_dscore"] < 1e-4


def test_large_batch_pair_kernel(B, oracle_mod):
    """16,384 queries (the C4 global batch) on 100K entries: 64 CTA-pair query tiles; sampled
    oracle parity plus the batch-wide properties."""
    n, b = 100_000, 16384
    emb, cl = synth.entries(n, seed=5001)
    g = B.NirvanaCache(entry_capacity=n, dim=768, latent_bytes=0, latent_capacity=5 * n)
    g.insert(torch.from_numpy(emb).cuda())
    q, _, _ = synth.queries(emb, cl, b, seed=5002)
    out = gpu_to_numpy(g.query(torch.from_numpy(q).cuda(), topk=1, latents=False))
    assert (out["ids"][:, 0] < n).all()
    o = oracle_mod.OracleCache(dim=768, entry_capacity=n, latent_bytes=0)
    o.insert(emb)
    rows = list(np.random.default_rng(5).choice(b, 254, replace=False)) + [0, b - 1]
    rep = check_batch(out, o, q, 1, rows=rows, adopt=False)
    print(rep)
    assert rep["max_dscore"] < 1e-4
