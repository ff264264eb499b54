"""Pins of the fp64 oracle against what the paper and mathematics fix (no GPU needed).

Each test checks the oracle against something other than itself: a cited paper / SPEC value
(tests/golden/), exact rational or 60-digit decimal arithmetic, a library routine (torch's
fp32->bf16 RNE), an independent integer re-derivation, or a brute-force property.
"""
import struct
from decimal import Decimal, getcontext
from fractions import Fraction

import numpy as np
import pytest

import synth
from tests.conftest import golden

getcontext().prec = 60


# ----------------------------------------------------------------------------------------
# bf16 rounding (reading R2)
# ----------------------------------------------------------------------------------------
def _bits_of(v: float) -> int:
    """bf16 bit pattern of a bf16-representable double (via its exact fp32 encoding)."""
    u = struct.unpack("<I", struct.pack("<f", v))[0]
    assert struct.unpack("<f", struct.pack("<I", u))[0] == v or v != v
    assert u & 0xFFFF == 0, f"{v!r} is not bf16-representable"
    return u >> 16


def _bf16_exact(v: float) -> float:
    """Independent re-derivation with exact rationals: nearest multiple of the bf16 quantum
    2^(E-7) (E = floor(log2|v|), quantum floored at 2^-133), ties to even (Fraction.__round__)."""
    if v == 0.0:
        return v
    x = Fraction(v)
    a = abs(x)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if Fraction(2) ** e > a:
        e -= 1
    q = max(e - 7, -133)
    m = round(x / Fraction(2) ** q)
    return float(m * Fraction(2) ** q)


def test_bf16_spot_values(oracle_mod):
    for a, bits in golden("bf16_spot_values.txt"):
        v = float.fromhex(a) if "0x" in a else float(a)
        got = oracle_mod.bf16_round(v)
        assert _bits_of(got) == int(bits, 16), (a, hex(_bits_of(got)), bits)


def test_bf16_vs_exact_rational_random(oracle_mod):
    rng = np.random.default_rng(1)
    vals = list(rng.standard_normal(3000) * np.exp2(rng.integers(-140, 5, 3000)))
    # exact midpoints and near-midpoints, normal and subnormal range
    for _ in range(1500):
        e = int(rng.integers(-140, 3))
        m = int(rng.integers(128, 256))
        q = max(e - 7, -133)
        mid = (m + 0.5) * 2.0 ** q if e >= -126 else (int(rng.integers(0, 128)) + 0.5) * 2.0 ** -133
        vals += [mid, np.nextafter(mid, 0), np.nextafter(mid, 10), -mid]
    for v in vals:
        v = float(v)
        assert oracle_mod.bf16_round(v) == _bf16_exact(v), v.hex()


def test_bf16_vs_torch_library_on_fp32_values(oracle_mod):
    """For fp32-representable inputs, fp64->bf16 RNE equals torch's fp32->bf16 RNE."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(2)
    f32 = (rng.standard_normal(20000) * np.exp2(rng.integers(-30, 3, 20000))).astype(np.float32)
    lib = torch.from_numpy(f32).to(torch.bfloat16).to(torch.float32).numpy()
    got = np.array([oracle_mod.bf16_round(float(v)) for v in f32])
    assert np.array_equal(got, lib.astype(np.float64))


# ----------------------------------------------------------------------------------------
# normalise: stored rows are the nearest bf16 values to the exact x/||x||  (R2)
# ----------------------------------------------------------------------------------------
def _exact_unit(x):
    xs = [Decimal(float(v)) for v in x]
    nrm = sum(v * v for v in xs).sqrt()
    return [v / nrm for v in xs]


@pytest.mark.parametrize("dim", [5, 64, 768])
def test_normalise_is_nearest_bf16_of_exact_unit_vector(oracle_mod, dim):
    rng = np.random.default_rng(dim)
    for trial in range(4):
        x = rng.standard_normal(dim).astype(np.float32) * np.float32(10.0 ** (trial - 2))
        st, y = oracle_mod.normalise(x.astype(np.float64))
        assert st == 0
        exact = _exact_unit(x)
        for yi, ei in zip(y, exact):
            assert _bits_of(float(yi)) >= 0  # bf16-representable
            err = abs(Decimal(float(yi)) - ei)
            # half a bf16 quantum at this magnitude (+ slack for fp64 norm rounding, 2^-40 rel)
            e = int(np.floor(np.log2(abs(float(ei))))) if ei != 0 else -200
            half_q = Decimal(2) ** (max(e - 7, -133) - 1)
            assert err <= half_q * (1 + Decimal(2) ** -30), (float(yi), float(ei))


def test_normalise_spec_example_and_errors(oracle_mod):
    x = np.zeros(64)
    x[0], x[1] = 3.0, 4.0           # (3,4,0,...) -> (0.6, 0.8)
    st, y = oracle_mod.normalise(x)
    assert st == 0 and _bits_of(y[0]) == 0x3F1A and _bits_of(y[1]) == 0x3F4D
    assert oracle_mod.normalise(np.zeros(8))[0] == oracle_mod.ROW_ZERO_NORM
    bad = np.ones(8)
    bad[3] = np.nan
    assert oracle_mod.normalise(bad)[0] == oracle_mod.ROW_NONFINITE
    bad[3] = np.inf
    assert oracle_mod.normalise(bad)[0] == oracle_mod.ROW_NONFINITE


# ----------------------------------------------------------------------------------------
# cosine + exact top-k (R1, R3) against 60-digit decimal brute force
# ----------------------------------------------------------------------------------------
def _exact_cos(a, b):
    da = [Decimal(float(v)) for v in a]
    db = [Decimal(float(v)) for v in b]
    dot = sum(x * y for x, y in zip(da, db))
    return dot / (sum(x * x for x in da).sqrt() * sum(y * y for y in db).sqrt())


@pytest.mark.parametrize("dim,n", [(64, 120), (768, 40)])
def test_query_topk_matches_decimal_brute_force(oracle_mod, dim, n):
    rng = np.random.default_rng(10 + dim)
    emb, cl = synth.entries(n, seed=3, dim=dim)
    emb[7] = emb[3]                       # exact duplicate -> tie broken by lower id (R3)
    o = oracle_mod.OracleCache(dim=dim, entry_capacity=n)
    rc, ids, st = o.insert(emb)
    assert rc == 0 and list(ids) == list(range(n))
    q, _, _ = synth.queries(emb, cl, 6, seed=5)
    q[0] = emb[3]
    topk = 5
    res = o.query(q, topk=topk, apply_counters=False)
    for r in range(q.shape[0]):
        _, qt = oracle_mod.normalise(q[r].astype(np.float64))
        exact = [(_exact_cos(qt, o.row(i)), i) for i in range(n)]
        exact.sort(key=lambda t: (-t[0], t[1]))
        for t in range(topk):
            gid = int(res["ids"][r, t])
            assert abs(Decimal(res["raw"][r, t]) - exact[t][0]) < Decimal("1e-13")
            # ranks agree unless two exact scores are within fp64 noise
            if t + 1 < n and exact[t][0] - exact[t + 1][0] > Decimal("1e-12") and \
                    (t == 0 or exact[t - 1][0] - exact[t][0] > Decimal("1e-12")):
                assert gid == exact[t][1]
    assert int(res["ids"][0, 0]) == 3 and int(res["ids"][0, 1]) == 7   # tie: lower id first
    assert res["raw"][0, 0] == res["raw"][0, 1]


def test_cosine_identities(oracle_mod):
    """SPEC S:66-70 (a==b -> 1, orthogonal -> 0, a,-a -> -1) and ||a-b||^2 = 2(1-s)."""
    d = 64
    e = np.zeros((3, d), dtype=np.float32)
    e[0, 0] = 1.0
    e[1, 1] = 1.0
    e[2, 0] = -1.0
    o = oracle_mod.OracleCache(dim=d, entry_capacity=8)
    o.insert(e)
    res = o.query(e[:1], topk=3, apply_counters=False)
    assert list(res["ids"][0]) == [0, 1, 2]
    assert list(res["raw"][0]) == [1.0, 0.0, -1.0]
    rng = np.random.default_rng(4)
    x = rng.standard_normal((2, d)).astype(np.float32)
    o2 = oracle_mod.OracleCache(dim=d, entry_capacity=8)
    o2.insert(x[1:])
    s = o2.query(x[:1], topk=1, apply_counters=False)["raw"][0, 0]
    _, a = oracle_mod.normalise(x[0].astype(np.float64))
    b = o2.row(0)
    a = a / np.sqrt(np.sum(a * a))
    b = b / np.sqrt(np.sum(b * b))
    assert abs(np.sum((a - b) ** 2) - 2 * (1 - s)) < 1e-12


# ----------------------------------------------------------------------------------------
# Fig. 11 map, holes, hand cache H
# ----------------------------------------------------------------------------------------
def test_fig11_truth_table(oracle_mod):
    o = oracle_mod.OracleCache(dim=8, entry_capacity=4)
    for s, k in golden("fig11_truth_table.txt"):
        assert o.select_k(float(s)) == int(k), s
    grid = np.linspace(-1, 1, 4001)
    ks = [o.select_k(float(s)) for s in grid]
    assert all(a <= b for a, b in zip(ks, ks[1:]))         # monotone in s


def test_knob_biases_one_bucket_up(oracle_mod):
    """k_bias (R20): hits move up by k_bias buckets (clamped), misses stay misses."""
    o = oracle_mod.OracleCache(dim=8, entry_capacity=4, k_bias=1)
    assert [o.select_k(s) for s in (0.60, 0.70, 0.80, 0.87, 0.92, 0.96)] == [0, 10, 15, 20, 25, 25]


def _kidx(k):
    return synth.K_VALUES.index(k)


def test_hole_rule_cases(oracle_mod):
    """Drive the hole rule through real queries: an entry u0-equivalent at exact cosine s."""
    H = synth.hand_vectors(16)
    # similarity -> K* : use the H pairs with known exact cosines
    sims = {25: (H[0], H[0]), 20: (H[0], H[4]), 15: (H[0], H[3]), 10: (H[2], H[3]),
            5: (H[0], H[1]), 0: (H[0], H[2])}
    for kstar, present, kused in golden("holes_cases.txt"):
        kstar, kused = int(kstar), int(kused)
        mask = 0 if present == "-" else sum(1 << _kidx(int(k)) for k in present.split(","))
        if mask == 0:
            continue       # an entry with no K is never stored (dirty); covered by evict tests
        qv, ev = sims[kstar]
        o = oracle_mod.OracleCache(dim=16, entry_capacity=4)
        rc, _, st = o.insert(ev[None, :], present=np.array([mask], dtype=np.uint8))
        assert rc == 0
        res = o.query(qv[None, :], topk=1)
        assert res["kstar"][0] == kstar
        assert res["k"][0] == kused, (kstar, present)


def test_hand_cache_H(oracle_mod):
    H = synth.hand_vectors(768)
    names = {f"u{i}": H[i] for i in range(5)}
    o = oracle_mod.OracleCache(dim=768, entry_capacity=8)
    o.insert(H[1:])                       # ids: u1=0, u2=1, u3=2, u4=3
    idmap = {"u1": 0, "u2": 1, "u3": 2, "u4": 3}
    for qn, en, s, k in golden("hand_cache_H.txt"):
        if en == "u0":
            continue
        assert o.score_id(names[qn], idmap[en]) == float(s)        # bit-exact
    r = o.query(H[[0, 2]], topk=4, apply_counters=False)
    assert list(r["ids"][0]) == [3, 2, 0, 1] and r["k"][0] == 20      # u4 > u3 > u1 > u2
    assert list(r["raw"][0]) == [0.9375, 0.875, 0.75, 0.5]
    assert r["ids"][1, 0] == 1 and r["raw"][1, 0] == 1.0 and r["k"][1] == 25   # u2 is cached
    o3 = oracle_mod.OracleCache(dim=768, entry_capacity=8)
    o3.insert(H[[1, 3, 4]])               # without u2: u2 -> u1 (0.875) -> K = 15
    r3 = o3.query(H[2:3], topk=3, apply_counters=False)
    assert list(r3["ids"][0]) == [0, 1, 2] and list(r3["raw"][0]) == [0.875, 0.8125, 0.71875]
    assert r3["k"][0] == 15
    # only u1 cached: s = 0.75 exactly -> the strict boundary of Fig. 11 -> K = 5
    o1 = oracle_mod.OracleCache(dim=768, entry_capacity=8)
    o1.insert(H[1:2])
    r1 = o1.query(H[:1], topk=1)
    assert r1["raw"][0, 0] == 0.75 and r1["k"][0] == 5
    # u0 itself -> 1.0 -> K=25; duplicate u4 (id 4) ties with u4 (id 3) -> id 3 wins
    o.insert(H[0:1])
    o.insert(H[4:5])
    r2 = o.query(H[[0, 4]], topk=2, apply_counters=False)
    assert r2["ids"][0, 0] == 4 and r2["k"][0] == 25
    assert list(r2["ids"][1]) == [3, 5] and r2["raw"][1, 0] == r2["raw"][1, 1] == 1.0
    # holes in H: u4 with {5,10,15}; query u0 -> K*=20 -> 15.  u4 with {25} only -> miss,
    # no fallback to u3 (R7)
    for mask, want in ((0b00111, 15), (0b10000, 0)):
        oh = oracle_mod.OracleCache(dim=768, entry_capacity=8)
        oh.insert(H[3:5], present=np.array([0b11111, mask], dtype=np.uint8))
        rr = oh.query(H[:1], topk=1)
        assert rr["ids"][0, 0] == 1 and rr["kstar"][0] == 20 and rr["k"][0] == want


# ----------------------------------------------------------------------------------------
# gather, counters, insert/evict (LCBFU) semantics
# ----------------------------------------------------------------------------------------
def test_gather_round_trip_and_counters(oracle_mod):
    L = 64
    emb, cl = synth.entries(50, seed=11, dim=64)
    lat = synth.latents_np(np.arange(50), 5, L, seed=11)
    o = oracle_mod.OracleCache(dim=64, entry_capacity=50, latent_bytes=L)
    o.insert(emb, latents=lat)
    q, anchor, _ = synth.queries(emb, cl, 40, seed=12)
    r = o.query(q, topk=1)
    hits = 0
    for i in range(40):
        if r["k"][i] > 0:
            hits += 1
            e = int(r["ids"][i, 0])
            assert np.array_equal(r["latents"][i], lat[e, _kidx(int(r["k"][i]))])  # bitwise
        else:
            assert not r["latents"][i].any()
    total = sum(int(o.meta(e)[0].sum()) for e in range(50))
    assert total == hits                   # one increment per hit (conservation)


def test_lcbfu_paper_example(oracle_mod):
    for k, f, score in golden("lcbfu_example.txt"):
        assert int(k) * int(f) == int(score)
    # Drive real counters: entry A holds only K=25 accessed 100x; entry B only K=5 accessed 200x.
    H = synth.hand_vectors(16)
    o = oracle_mod.OracleCache(dim=16, entry_capacity=4)
    o.insert(H[[0, 2]], present=np.array([1 << 4, 1 << 0], dtype=np.uint8))
    o.record_access(np.zeros(100, np.uint64), np.full(100, 25, np.int32))
    o.record_access(np.ones(200, np.uint64), np.full(200, 5, np.int32))
    rc, ev, dirty = o.evict(1)
    assert rc == 0 and list(ev) == [(1 << 3) | 0]          # the K=5 item (score 1000) goes first
    assert list(dirty) == [1] and o.live_entries == 1     # its only K -> dirty


def test_evict_optimality_fuzz(oracle_mod):
    """Evicted keys <= every surviving key (acceptance #5), checked by exhaustive scan."""
    rng = np.random.default_rng(21)
    emb, _ = synth.entries(60, seed=21, dim=16)
    pres = synth.present_masks(60, seed=21, hole_frac=0.3)
    o = oracle_mod.OracleCache(dim=16, entry_capacity=60)
    o.insert(emb, present=pres)
    for _ in range(300):
        live = [e for e in range(60) if _live(o, e)]
        e = int(rng.choice(live))
        f, m = o.meta(e)
        js = [j for j in range(5) if m >> j & 1]
        o.record_access(np.array([e], np.uint64), np.array([synth.K_VALUES[int(rng.choice(js))]], np.int32))
    for n in (7, 1, 33, 0):
        before = {}
        for e in range(60):
            if _live(o, e):
                f, m = o.meta(e)
                for j in range(5):
                    if m >> j & 1:
                        before[(e, j)] = (int(f[j]) * synth.K_VALUES[j], e, j)
        rc, ev, dirty = o.evict(n)
        assert rc == 0 and len(ev) == n
        gone = {(int(x) >> 3, int(x) & 7) for x in ev}
        survivors = [v for k, v in before.items() if k not in gone]
        if gone and survivors:
            assert max(before[g] for g in gone) < min(survivors)
        keys = [before[g] for g in [(int(x) >> 3, int(x) & 7) for x in ev]]
        assert keys == sorted(keys)                         # reported in eviction order
        for d in dirty:                                     # dirty completeness
            assert all(before.get((int(d), j)) is None or (int(d), j) in gone for j in range(5))
    assert o.evict(o.live_items + 1)[0] == oracle_mod.E_EVICT_RANGE


def _live(o, e):
    try:
        o.meta(e)
        return True
    except KeyError:
        return False


def test_insert_full_and_bad_rows(oracle_mod):
    emb, _ = synth.entries(6, seed=1, dim=16)
    o = oracle_mod.OracleCache(dim=16, entry_capacity=4, latent_capacity=12)
    bad = emb.copy()
    bad[1] = 0.0
    bad[2, 3] = np.inf
    rc, ids, st = o.insert(bad[:4])
    assert rc == 0 and list(st) == [0, 2, 1, 0] and ids[1] == oracle_mod.NO_ID and list(ids[[0, 3]]) == [0, 1]
    assert o.insert(emb[:3])[0] == oracle_mod.E_FULL and o.live_entries == 2   # S:246, no change
    assert o.insert(emb[:2], present=np.array([1, 1], np.uint8))[0] == 0       # 10 + 2 items fit
    assert o.insert(emb[:1])[0] == oracle_mod.E_FULL
    r = o.query(np.vstack([emb[:1], np.zeros((1, 16), np.float32)]), topk=1)
    assert r["rc"] == oracle_mod.E_BAD_ROWS and list(r["status"]) == [0, 2] and r["k"][1] == 0


def test_empty_cache_is_a_miss(oracle_mod):
    o = oracle_mod.OracleCache(dim=16, entry_capacity=4)
    r = o.query(np.ones((2, 16), np.float32), topk=3)
    assert (r["ids"] == oracle_mod.NO_ID).all() and (r["k"] == 0).all() and np.isneginf(r["scores"]).all()
