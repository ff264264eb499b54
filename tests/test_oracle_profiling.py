"""Pins of the oracle's cache-selector profiling (Alg. 2; reading R25)."""
import numpy as np

import synth
from oracle import profiling


def _hand(oracle_mod):
    """Cache = {u1}; profiling prompts u0, u2, u4 -> exact similarities 0.75, 0.875, 0.921875
    (dyadic components: every product and sum exact)."""
    H = synth.hand_vectors(16)
    o = oracle_mod.OracleCache(dim=16, entry_capacity=4)
    o.insert(H[[1]])
    return o, H[[0, 2, 4]]


def test_hand_profile_exact(oracle_mod):
    o, q = _hand(oracle_mod)
    sims = o.query(q, topk=1, want_latents=False, apply_counters=False)["scores"][:, 0]
    assert list(sims) == [0.75, 0.875, 0.921875]
    #            u0   u2   u4       (quality per prompt; alpha = 0.9)
    quality = np.array([[0.95, 0.97, 0.99],    # K=5  : all pass -> smallest similarity 0.75
                        [0.50, 0.95, 0.99],    # K=10 : u0 fails -> 0.75
                        [0.50, 0.80, 0.99],    # K=15 : u0, u2 fail -> 0.875
                        [0.10, 0.20, 0.90],    # K=20 : all fail (0.90 is not > 0.9) -> 0.921875
                        [0.10, 0.20, 0.30]])   # K=25 : all fail -> 0.921875
    thr, failed = profiling.profile_thresholds(o, q, quality, 0.9)
    assert list(thr) == [0.75, 0.75, 0.875, 0.921875, 0.921875]
    assert list(failed) == [False, True, True, True, True]


def test_monotone_repair(oracle_mod):
    """A K whose own worst failure is lower than a smaller K's threshold inherits it."""
    o, q = _hand(oracle_mod)
    quality = np.array([[0.5, 0.8, 0.99], [0.5, 0.99, 0.99], [0.99] * 3, [0.99] * 3, [0.99] * 3])
    thr, _ = profiling.profile_thresholds(o, q, quality, 0.9)
    assert list(thr) == [0.875, 0.875, 0.875, 0.875, 0.875]


def test_definition_by_brute_force(oracle_mod):
    """Random cache / prompts / qualities: for each K the threshold is a profiled similarity of
    a failing image and every image strictly above it passed (checked before the monotone
    repair by recomputing from the similarities)."""
    rng = np.random.default_rng(0)
    emb, cl = synth.entries(300, seed=9, dim=32)
    o = oracle_mod.OracleCache(dim=32, entry_capacity=300)
    o.insert(emb)
    q, _, _ = synth.queries(emb, cl, 80, seed=10)
    quality = rng.random((5, 80))
    thr, failed = profiling.profile_thresholds(o, q, quality, 0.5)
    sims = o.query(q, topk=1, want_latents=False, apply_counters=False)["scores"][:, 0]
    prev = -np.inf
    for j in range(5):
        fails = sims[quality[j] <= 0.5]
        raw = fails.max() if fails.size else sims.min()
        assert (quality[j][sims > raw] > 0.5).all()
        if fails.size:
            assert raw in sims[quality[j] <= 0.5]
        prev = max(prev, raw)
        assert thr[j] == prev and failed[j] == bool(fails.size)


def test_recovers_fig11_table_from_its_quality_model(oracle_mod):
    """A quality model whose K-th curve crosses alpha exactly at the paper's Fig. 11 threshold
    (quality(s, K) = alpha + (s - tau_K)): profiling prompts spanning the similarity range give
    back tau_K from below, to within the spacing of the profiled similarities."""
    tau = np.array([0.65, 0.75, 0.85, 0.90, 0.95])
    emb, cl = synth.entries(400, seed=21, dim=64)
    o = oracle_mod.OracleCache(dim=64, entry_capacity=400)
    o.insert(emb)
    q, _, _ = synth.queries(emb, cl, 600, seed=22)
    sims = o.query(q, topk=1, want_latents=False, apply_counters=False)["scores"][:, 0]
    quality = 0.9 + (sims[None, :] - tau[:, None])
    thr, failed = profiling.profile_thresholds(o, q, quality, 0.9)
    assert failed.all()
    for j in range(5):
        below = sims[sims <= tau[j]]
        assert thr[j] == below.max() and tau[j] - thr[j] < 0.02
