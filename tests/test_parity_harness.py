"""The parity harness itself (tests/parity.py) on CPU: a GPU result that is the oracle's own
answer passes, and each plausible kernel bug -- a dropped or swapped rank 2..k candidate, a
wrong score, a wrong K, a stored component rounded the wrong way -- fails.  Also pins the
stored-row accept set on a row whose quotient is an exact bf16 midpoint."""
import numpy as np
import pytest

import synth
from tests.parity import NO_ID, check_batch, check_stored_row


def _cache(oracle_mod, n=400, seed=31):
    emb, cl = synth.entries(n, seed=seed, dim=64)
    o = oracle_mod.OracleCache(dim=64, entry_capacity=n, latent_bytes=0)
    o.insert(emb)
    q, _, _ = synth.queries(emb, cl, 24, seed=seed + 1)
    return o, emb, q


def _as_gpu(o, q, topk):
    r = o.query(q, topk=topk, want_latents=False, apply_counters=False)
    return dict(ids=r["ids"].copy(), scores=r["scores"].astype(np.float32), k=r["k"].copy(), latents=None)


def _separated_row(o, q, topk, rank):
    """A query row whose oracle gaps around `rank` exceed 2e-3 on both sides."""
    r = o.query(q, topk=topk + 1, want_latents=False, apply_counters=False)
    for i in range(q.shape[0]):
        s = r["raw"][i]
        if s[rank - 1] - s[rank] > 2e-3 and s[rank] - s[rank + 1] > 2e-3:
            return i
    pytest.skip("no well-separated row in this sample")


def test_oracle_answer_passes(oracle_mod):
    o, _, q = _cache(oracle_mod)
    for topk in (1, 4, 16):
        rep = check_batch(_as_gpu(o, q, topk), o, q, topk, adopt=False)
        assert rep["ranks_checked"] == q.shape[0] * topk and rep["max_dscore"] < 1e-6


def test_swapped_lower_ranks_fail(oracle_mod):
    o, _, q = _cache(oracle_mod)
    g = _as_gpu(o, q, 4)
    i = _separated_row(o, q, 4, 2)
    g["ids"][i, [2, 3]] = g["ids"][i, [3, 2]]
    g["scores"][i, [2, 3]] = g["scores"][i, [3, 2]]
    with pytest.raises(AssertionError):
        check_batch(g, o, q, 4, adopt=False)


def test_dropped_third_best_fails(oracle_mod):
    """A kernel that loses the true 3rd-best and reports the 4th and 5th in its place."""
    o, _, q = _cache(oracle_mod)
    g = _as_gpu(o, q, 4)
    i = _separated_row(o, q, 4, 2)
    full = o.query(q[i:i + 1], topk=5, want_latents=False, apply_counters=False)
    g["ids"][i, 2:] = full["ids"][0, 3:5]
    g["scores"][i, 2:] = full["scores"][0, 3:5]
    with pytest.raises(AssertionError):
        check_batch(g, o, q, 4, adopt=False)


def test_wrong_score_k_and_padding_fail(oracle_mod):
    o, _, q = _cache(oracle_mod)
    g = _as_gpu(o, q, 2)
    g["scores"][3, 1] -= 3e-4
    with pytest.raises(AssertionError):
        check_batch(g, o, q, 2, adopt=False)
    g = _as_gpu(o, q, 2)
    hit = int(np.nonzero(g["k"] > 0)[0][0])
    g["k"][hit] = 25 if g["k"][hit] != 25 else 5
    with pytest.raises(AssertionError):
        check_batch(g, o, q, 2, adopt=False)
    g = _as_gpu(o, q, 2)
    g["ids"][0, 1] = NO_ID                                        # a missing rank-2 entry
    with pytest.raises(AssertionError):
        check_batch(g, o, q, 2, adopt=False)


def _midpoint_row(dim=64):
    """A row with ||x|| = 1 exactly whose first component is the bf16 rounding midpoint
    0.5 + 2^-9 (between 0.5 and 0.50390625): the rest is 1 - x0^2 written as a sum of squares
    of powers of two (each power of two is 4^k or 2 * 4^k), so every sum is exact."""
    x0 = 0.5 + 2.0 ** -9
    rest = 1.0 - x0 * x0              # exact dyadic
    comps = []
    for e in range(0, -60, -1):
        if rest >= 2.0 ** e:
            rest -= 2.0 ** e
            if e % 2 == 0:
                comps.append(2.0 ** (e // 2))
            else:
                comps += [2.0 ** ((e - 1) // 2)] * 2
    assert rest == 0.0 and len(comps) < dim
    x = np.zeros(dim)
    x[0] = x0
    x[1:1 + len(comps)] = comps
    assert np.sum(x * x) == 1.0
    return x


def test_stored_row_accept_set(oracle_mod):
    x = _midpoint_row()
    st, y = oracle_mod.normalise(x)
    assert st == 0 and y[0] == 0.5                              # RNE: the even neighbour
    bits = (y.astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
    assert check_stored_row(bits, x, y) == 0
    other = bits.copy()
    other[0] += 1                                                # 0.50390625: the odd neighbour
    assert check_stored_row(other, x, y) == 1                    # provably a midpoint case
    wrong = bits.copy()
    wrong[2] += 1                                                # not near a midpoint
    with pytest.raises(AssertionError):
        check_stored_row(wrong, x, y)
    far = bits.copy()
    far[0] += 2                                                  # not adjacent
    with pytest.raises(AssertionError):
        check_stored_row(far, x, y)
