"""The fused eviction (evict.cu: one cooperative launch selects the exact n smallest unit keys
and applies them, readings R11-R13, R24) against the oracle, on every path the
selection can take: compaction after the first linear level (the common case), late or no
compaction (forced through the candidate-buffer cap), selection finished at level 0, n = 1,
n = every live unit, heavy-hitter counters whose keys spread over many log bins; plus the
sorts the eviction lists go through (one-CTA bitonic, LSD over a narrow key range)."""
import numpy as np
import pytest
import torch

import synth
from tests.parity import check_batch, gpu_to_numpy

pytestmark = pytest.mark.gpu
L = 64


@pytest.mark.parametrize("n", [1, 2, 3, 1000, 4097, 16384])
def test_small_sort(n):
    from paper_2312_04429_b200 import binding as B
    rng = np.random.default_rng(n)
    k = rng.integers(0, 2**63, n, dtype=np.int64).view(np.uint64) * np.uint64(2)
    k[: n // 3] = k[0]   # duplicates
    t = torch.from_numpy(k.view(np.int64).copy()).cuda()
    B.debug_sort_u64_ex(t, small=True)
    assert np.array_equal(t.cpu().numpy().view(np.uint64), np.sort(k))


@pytest.mark.parametrize("coop", [0, 2])
@pytest.mark.parametrize("n", [2, 20_000, 300_001])
@pytest.mark.parametrize("bits", [1, 9, 23, 40])
def test_range_sort(n, bits, coop):
    from paper_2312_04429_b200 import binding as B
    rng = np.random.default_rng(bits)
    base = np.uint64(123456789) << np.uint64(20)
    k = base + (rng.integers(0, 2**bits, n, dtype=np.int64).astype(np.uint64))
    t = torch.from_numpy(k.view(np.int64).copy()).cuda()
    B.debug_sort_u64_ex(t, bits=bits, base=int(base), small=coop)
    assert np.array_equal(t.cpu().numpy().view(np.uint64), np.sort(k))


def _pair(oracle_mod, n, policy, gran, seed, nq_batches=3, zipf_hot=False):
    from paper_2312_04429_b200 import binding as B
    emb, cl = synth.entries(n, seed=seed)
    pres = synth.present_masks(n, seed=seed, hole_frac=0.2)
    lat = synth.latents_np(np.arange(n), 5, L, seed=seed)
    g = B.NirvanaCache(entry_capacity=n + 64, latent_capacity=5 * n + 64, dim=768, latent_bytes=L,
                       evict_granularity=gran)
    g.set_evict_policy(policy)
    o = oracle_mod.OracleCache(dim=768, entry_capacity=n + 64, latent_capacity=5 * n + 64, latent_bytes=L)
    g.insert(torch.from_numpy(emb).cuda(), torch.from_numpy(lat).cuda(), present=pres)
    o.insert(emb, latents=lat, present=pres)
    for r in range(nq_batches):
        if zipf_hot:   # the same few prompts again and again: counters / clocks far apart
            q = np.repeat(emb[(np.arange(64) * 7) % n], 4, axis=0)
        else:
            q, _, _ = synth.queries(emb, cl, 256, seed=seed * 100 + r)
        _query_both(g, o, q)
    return B, g, o


def _query_both(g, o, q):
    """One batch on both sides; the harness makes the oracle adopt the GPU's accepted
    (entry, K) on near-ties so the counters / clocks stay equal."""
    out = gpu_to_numpy(g.query(torch.from_numpy(np.ascontiguousarray(q, dtype=np.float32)).cuda(), topk=1))
    check_batch(out, o, q, 1, expected_latent=None)


def _evict_both(B, g, o, n, policy, gran):
    if gran:
        ev, dirty = g.evict(n)
        rc, oev = o.evict_entries(n, policy=policy)
        assert rc == 0
        assert np.array_equal(ev, oev)
        assert np.array_equal(np.sort(dirty), np.sort(oev))
    else:
        ev, dirty = g.evict(n)
        rc, oev, od = o.evict(n, policy=policy)
        assert rc == 0
        assert np.array_equal(ev, oev)
        assert np.array_equal(dirty, od)
    return B.debug_evict_stats(g)


@pytest.mark.parametrize("gran", [0, 1])
@pytest.mark.parametrize("policy", [0, 1, 2, 3])
@pytest.mark.parametrize("cap", [-1, 0, 1, 37, 5000])
def test_fused_evict_paths(oracle_mod, policy, gran, cap):
    """Rounds of query / evict with the candidate buffer capped: cap 0 never compacts (the
    level sweeps and the apply run over the slot columns), small caps compact late."""
    B, g, o = _pair(oracle_mod, 1500, policy, gran, seed=70 + policy, zipf_hot=(policy in (0, 2)))
    B.debug_set_evict_cand_cap(g, cap)
    B.debug_evict_window(g, 0)   # the two-sweep path (the window has its own test)
    rng = np.random.default_rng(policy * 10 + gran)
    for rnd in range(4):
        units = g.evict_units
        n = int(rng.integers(1, max(2, units // 3)))
        st = _evict_both(B, g, o, n, policy, gran)
        if cap == 0:
            assert st["compact_level"] == 0
        _query_both(g, o, np.asarray(synth.entries(32, seed=500 + rnd)[0]))


@pytest.mark.parametrize("gran", [0, 1])
@pytest.mark.parametrize("policy", [0, 1, 2, 3])
@pytest.mark.parametrize("stride", [1, 3, -1])
def test_single_sweep_window(oracle_mod, policy, gran, stride):
    """The single-sweep window: stride 1 samples every slot (the estimate is exact, so the
    selection always finishes on the level-0 candidates), 3 every third slot, -1 the automatic
    stride.  Every outcome must evict exactly what the oracle evicts."""
    B, g, o = _pair(oracle_mod, 1500, policy, gran, seed=170 + policy, zipf_hot=(policy in (0, 2)))
    B.debug_evict_window(g, stride)
    rng = np.random.default_rng(policy * 10 + gran + stride % 7)
    for rnd in range(4):
        units = g.evict_units
        n = int(rng.integers(1, max(2, units // 3)))
        _evict_both(B, g, o, n, policy, gran)
        w = B.debug_evict_window(g)
        assert w in (0, 1, 2)
        if stride == 1:
            assert w == 1, (rnd, n)
        _query_both(g, o, np.asarray(synth.entries(32, seed=600 + rnd)[0]))


@pytest.mark.parametrize("gran", [0, 1])
def test_single_sweep_window_missed(oracle_mod, gran):
    """An estimate that must miss: with stride 7 the sample is every 7th block of 32 slots; those
    blocks hold never-accessed items, every other slot items with f > 0, and a third of the
    units go -- the sample places the n-th key among the f = 0 keys while it lies far above them.
    The kernel sees that the n-th key's bin ends beyond the window and takes the two-sweep path;
    the eviction stays exact."""
    from paper_2312_04429_b200 import binding as B
    n = 1400
    emb, _ = synth.entries(n, seed=177)
    pres = synth.present_masks(n, seed=177, hole_frac=0.2)
    g = B.NirvanaCache(entry_capacity=n, latent_capacity=5 * n, dim=768, latent_bytes=0, evict_granularity=gran)
    o = oracle_mod.OracleCache(dim=768, entry_capacity=n, latent_capacity=5 * n)
    g.insert(torch.from_numpy(emb).cuda(), None, present=pres)
    o.insert(emb, present=pres)
    rng = np.random.default_rng(gran)
    for id_ in range(n):
        if (B.debug_slot_of(g, id_) // 32) % 7 == 0:
            continue
        for j in range(5):
            if (int(pres[id_]) >> j) & 1:
                f = int(rng.integers(1, 50))
                B.debug_set_count(g, id_, j, f)
                assert o.set_count(id_, j, f) == 0
    B.debug_evict_window(g, 7)
    nev = g.evict_units // 3
    if gran:
        ev, _ = g.evict(nev)
        rc, oev = o.evict_entries(nev)
        assert rc == 0 and np.array_equal(ev, oev)
    else:
        ev, dirty = g.evict(nev)
        rc, oev, od = o.evict(nev)
        assert rc == 0 and np.array_equal(ev, oev) and np.array_equal(dirty, od)
    assert B.debug_evict_window(g) == 2


@pytest.mark.parametrize("gran", [0, 1])
def test_fused_evict_extremes(oracle_mod, gran):
    """n = 1, then nearly everything, then every remaining unit."""
    B, g, o = _pair(oracle_mod, 800, 0, gran, seed=91, zipf_hot=True)
    _evict_both(B, g, o, 1, 0, gran)
    _evict_both(B, g, o, g.evict_units - 3, 0, gran)
    _evict_both(B, g, o, g.evict_units, 0, gran)
    assert g.evict_units == 0
    assert g.stats()["live_entries"] == 0


def test_fused_evict_hot_counters_spread(oracle_mod):
    """LCBFU with heavy hitters: the keys of accessed items spread over many log bins, and the
    cut falls among them when almost everything goes."""
    B, g, o = _pair(oracle_mod, 2000, 0, 0, seed=93, nq_batches=6, zipf_hot=True)
    units = g.evict_units
    st = _evict_both(B, g, o, units - 40, 0, 0)
    assert st["levels"] >= 1


def test_key_saturation_reading_r11(oracle_mod):
    """R11: the GPU item key saturates the LCBFU score f*K at 2^29 - 1.  (1) A cut below the
    saturated items gives exactly the oracle's eviction; (2) a cut AMONG them orders the
    saturated items by (id, K) on the GPU and by their exact f*K in the oracle -- the documented
    deviation, which needs > 5.4e8 / K accesses of one item to arise."""
    B, g, o = _pair(oracle_mod, 200, 0, 0, seed=95, nq_batches=0)
    picks = []
    for id_ in range(5, 200):
        _, mask = g.meta(id_)
        j = 4 if (mask >> 4) & 1 else (0 if mask & 1 else None)
        if j is not None:
            picks.append((id_, j))
        if len(picks) == 3:
            break
    kvals = (5, 10, 15, 20, 25)
    # exact f*K all > 2^29 - 1, DEcreasing with the id: the two orders then disagree
    fs = [-(-t // kvals[j]) for t, (_, j) in zip((4_000_000_000, 3_000_000_000, 2_000_000_000), picks)]
    for (i, j), f in zip(picks, fs):
        B.debug_set_count(g, i, j, f)
        assert o.set_count(i, j, f) == 0
    _evict_both(B, g, o, g.evict_units - 3, 0, 0)          # (1) identical
    exact = sorted(picks, key=lambda p: (fs[picks.index(p)] * kvals[p[1]], p[0], p[1]))
    ev, _ = g.evict(1)
    rc, oev, _ = o.evict(1)
    assert rc == 0
    assert int(ev[0]) == (min(picks)[0] << 3 | min(picks)[1])           # GPU: (id, j) among the saturated
    assert int(oev[0]) == (exact[0][0] << 3 | exact[0][1])               # oracle: exact f*K
    assert int(ev[0]) != int(oev[0])


@pytest.mark.parametrize("gran", [0, 1])
def test_evict_view_and_keys(oracle_mod, gran):
    """cache_evict_view hands out the same lists as cache_evict (in the library's pinned
    staging, no copy); cache_last_evicted_keys returns the full keys of that eviction, whose
    masked values are the list, ascending."""
    B, g, o = _pair(oracle_mod, 1200, 0, gran, seed=97, zipf_hot=True)
    ev, dirty = g.evict(g.evict_units // 5, view=True)
    if gran:
        rc, oev = o.evict_entries(len(ev))
        assert np.array_equal(ev, oev) and np.array_equal(dirty, np.sort(oev))
    else:
        rc, oev, od = o.evict(len(ev))
        assert np.array_equal(ev, oev) and np.array_equal(dirty, od)
    keys = g.last_evicted_keys()
    mask = np.uint64(0xFFFFFFFF) if gran else np.uint64((1 << 35) - 1)
    assert len(keys) == len(ev) and np.all(np.diff(keys.astype(np.float64)) >= 0)
    assert np.array_equal(keys & mask, ev)


@pytest.mark.parametrize("world,push", [(2, True), (3, False), (4, True)])
@pytest.mark.parametrize("policy,gran", [(0, 0), (1, 0), (2, 1), (3, 0)])
@pytest.mark.parametrize("cap", [-1, 0, 13])
def test_distributed_levels_equal_single_cache(world, push, policy, gran, cap):
    """The distributed fused eviction (cache_evict_sel_*: the levels with the histograms summed
    over ranks, by peer memory or by the caller) evicts exactly what one cache evicts, in the
    same order, under every policy / granularity and with the candidate buffer capped (0: the
    levels sweep the shards in full)."""
    from paper_2312_04429_b200 import binding as B, sharded as S
    n = 1500
    emb, cl = synth.entries(n, seed=31 + world)
    pres = synth.present_masks(n, seed=31, hole_frac=0.2)
    kw = dict(dim=768, latent_bytes=0, evict_granularity=gran)
    single = B.NirvanaCache(entry_capacity=n + 64, **kw)
    vs = S.VirtualShards(world, entry_capacity=n + 64, push_max_nb=(256 if push else 0), push_max_topk=1, **kw)
    for c in (single, vs):
        c.set_evict_policy(policy)
        c.insert(torch.from_numpy(emb).cuda(), None, present=pres)
    for c in vs.caches:
        B.debug_set_evict_cand_cap(c, cap)
    rng = np.random.default_rng(world * 7 + policy)
    for r in range(3):
        q = torch.from_numpy(synth.queries(emb, cl, 128 * world, seed=400 + r)[0]).cuda()
        a = single.query(q, latents=False)
        b = vs.query(q, latents=False)
        assert torch.equal(a["ids"], b["ids"]) and torch.equal(a["k"], b["k"])
        units = single.evict_units
        nev = int(rng.integers(1, max(2, units // 3)))
        e1, d1 = single.evict(nev)
        e2, d2 = vs.evict(nev)
        assert np.array_equal(e1, e2) and np.array_equal(d1, d2), (r, nev)
        # each rank's single-sweep window (level 0 compacts below its own estimate): held or
        # missed per rank, never when the candidate buffer is capped below the share
        wins = [B.debug_evict_window(c) for c in vs.caches]
        allowed = {-1: (1, 2), 0: (0,)}.get(cap, (0, 1, 2))
        assert all(w in allowed for w in wins), (wins, cap)
        ne, _ = synth.entries(40, seed=700 + r)
        single.insert(torch.from_numpy(ne).cuda())
        vs.insert(torch.from_numpy(ne).cuda())


def test_radix8_protocol_still_equal(oracle_mod):
    """Round 1's 8-pass radix protocol (kept selectable) against one cache."""
    from paper_2312_04429_b200 import binding as B, sharded as S
    n = 900
    emb, cl = synth.entries(n, seed=47)
    single = B.NirvanaCache(entry_capacity=n, dim=768, latent_bytes=0)
    for push in (True, False):
        vs = S.VirtualShards(3, entry_capacity=n, dim=768, latent_bytes=0, push_max_nb=(128 if push else 0))
        vs.evict_protocol = "radix8"
        s1 = B.NirvanaCache(entry_capacity=n, dim=768, latent_bytes=0)
        for c in (s1, vs):
            c.insert(torch.from_numpy(emb).cuda())
        q = torch.from_numpy(synth.queries(emb, cl, 384, seed=48)[0]).cuda()
        s1.query(q, latents=False)
        vs.query(q, latents=False)
        e1, d1 = s1.evict(777)
        e2, d2 = vs.evict(777)
        assert np.array_equal(e1, e2) and np.array_equal(d1, d2)


@pytest.mark.parametrize("policy,gran", [(0, 0), (1, 0), (0, 1)])
def test_fused_evict_parity_1m_entries(oracle_mod, policy, gran):
    """At scale: 1M entries (4.75M items; dim 64 so the fp64 oracle holds the cache), Zipf query
    batches (every row checked against the oracle, accesses adopted), then 1% and 5% evictions
    (items, or entries in entry mode): the fused eviction's lists equal the oracle's exactly
    (ids, order, dirty entries); the 1% eviction takes the single-sweep window."""
    from paper_2312_04429_b200 import binding as B
    n, dim = 1_000_000, 64
    emb, cl = synth.entries(n, seed=303, dim=dim)
    pres = synth.present_masks(n, seed=303)
    g = B.NirvanaCache(entry_capacity=n, latent_capacity=5 * n, dim=dim, latent_bytes=0, evict_granularity=gran)
    g.set_evict_policy(policy)
    o = oracle_mod.OracleCache(dim=dim, entry_capacity=n, latent_capacity=5 * n)
    for s0 in range(0, n, 200_000):
        g.insert(torch.from_numpy(emb[s0:s0 + 200_000]).cuda(), None, present=pres[s0:s0 + 200_000])
        o.insert(emb[s0:s0 + 200_000], present=pres[s0:s0 + 200_000])
    for r in range(3):
        q, _, _ = synth.queries(emb, cl, 256, seed=310 + r)
        _query_both(g, o, q)
    for frac in (0.01, 0.05):
        nev = int(g.evict_units * frac)
        ev, dirty = g.evict(nev)
        if gran:
            rc, oev = o.evict_entries(nev, policy=policy)
            assert rc == 0 and np.array_equal(ev, oev) and np.array_equal(dirty, np.sort(oev)), frac
        else:
            rc, oev, od = o.evict(nev, policy=policy)
            assert rc == 0 and np.array_equal(ev, oev) and np.array_equal(dirty, od), frac
        st = B.debug_evict_stats(g)
        assert st["full_sweeps"] <= 3
        if frac == 0.01:   # the single-sweep window holds the cut: one full sweep
            assert B.debug_evict_window(g) == 1 and st["full_sweeps"] == 1, st


def test_distributed_calls_out_of_order_fail_cleanly():
    """cache_evict_sel_*: levels out of order, a pick without its level, an apply without a
    selection -> CACHE_E_STATE, and the cache keeps working afterwards."""
    from paper_2312_04429_b200 import binding as B
    n = 600
    emb, _ = synth.entries(n, seed=61)
    g = B.NirvanaCache(entry_capacity=n, dim=768, latent_bytes=0)
    g.insert(torch.from_numpy(emb).cuda())
    h = torch.zeros(4096, dtype=torch.int32, device="cuda")
    with pytest.raises(B.CacheError) as ei:
        g.evict_sel_apply(10)                       # nothing begun
    assert ei.value.code == B.E_STATE
    g.evict_sel_begin(100)
    with pytest.raises(B.CacheError) as ei:
        g.evict_sel_level(1, h)                     # level 0 first
    assert ei.value.code == B.E_STATE
    with pytest.raises(B.CacheError) as ei:
        g.push_evict_sel_level(0)                   # no push arenas
    assert ei.value.code == B.E_STATE
    g.evict_sel_level(0, h)
    assert int(h.sum()) == g.live_items            # level 0 counts every live unit
    with pytest.raises(B.CacheError) as ei:
        g.evict_sel_apply(100)                      # picks not finished: nothing applied
    assert ei.value.code == B.E_STATE
    done = g.evict_sel_pick(0, h)
    lvl = 1
    while not done:
        g.evict_sel_level(lvl, h)
        done = g.evict_sel_pick(lvl, h)
        lvl += 1
    ev, dirty = g.evict_sel_apply(100)
    ref = B.NirvanaCache(entry_capacity=n, dim=768, latent_bytes=0)
    ref.insert(torch.from_numpy(emb).cuda())
    e2, d2 = ref.evict(100)
    assert np.array_equal(ev, e2) and np.array_equal(dirty, d2)
    assert len(g.evict(50)[0]) == 50                # the single-cache path still works


@pytest.mark.parametrize("dist", ["plateau", "geometric", "huge", "mixed"])
@pytest.mark.parametrize("gran", [0, 1])
def test_fused_evict_adversarial_counters(oracle_mod, dist, gran):
    """Counters set directly (both sides) to distributions the query streams never produce: one
    big plateau of equal scores (the level-0 log bin holds almost everything), geometric spreads,
    scores near the key's saturation, and a mix -- then evictions of random sizes under LCBFU and
    LFU: the selection must still be exact (order and dirty lists)."""
    from paper_2312_04429_b200 import binding as B
    n = 2500
    emb, _ = synth.entries(n, seed=500 + gran)
    pres = synth.present_masks(n, seed=500, hole_frac=0.3)
    rng = np.random.default_rng({"plateau": 1, "geometric": 2, "huge": 3, "mixed": 4}[dist] * 10 + gran)
    for policy in (0, 2):
        g = B.NirvanaCache(entry_capacity=n, latent_capacity=5 * n, dim=768, latent_bytes=0, evict_granularity=gran)
        g.set_evict_policy(policy)
        o = oracle_mod.OracleCache(dim=768, entry_capacity=n, latent_capacity=5 * n)
        g.insert(torch.from_numpy(emb).cuda(), None, present=pres)
        o.insert(emb, present=pres)
        for id_ in range(n):
            for j in range(5):
                if not (int(pres[id_]) >> j) & 1:
                    continue
                if dist == "plateau":
                    f = 3 if rng.random() < 0.9 else int(rng.integers(0, 6))
                elif dist == "geometric":
                    f = int(rng.geometric(0.05)) - 1
                elif dist == "huge":
                    f = int(rng.integers(0, 40_000_000))   # f * K up to 1e9: beyond the 2^29 - 1 key cap
                else:
                    f = int(rng.choice([0, 1, 7, 1000, 123456]))
                if dist == "huge" and policy == 0:
                    f = min(f, (2 ** 29 - 1) // (5 * (j + 1)))   # keep LCBFU below the cap (R11 is tested apart)
                if f:
                    B.debug_set_count(g, id_, j, f)
                    assert o.set_count(id_, j, f) == 0
        for _ in range(3):
            units = g.evict_units
            if units < 2:
                break
            nev = int(rng.integers(1, units))
            if gran:
                ev, dirty = g.evict(nev)
                rc, oev = o.evict_entries(nev, policy=policy)
                assert rc == 0 and np.array_equal(ev, oev), (dist, policy)
            else:
                ev, dirty = g.evict(nev)
                rc, oev, od = o.evict(nev, policy=policy)
                assert rc == 0 and np.array_equal(ev, oev) and np.array_equal(dirty, od), (dist, policy)
