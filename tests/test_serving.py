"""NEXT-1: the Alg. 1 serving loop's accounting against the paper's formulas (CPU; the cache
is played by the fp64 oracle through an adapter -- test infrastructure)."""
import math

import numpy as np
import pytest

import synth
from paper_2312_04429_b200.serving import (LatencyParams, RunReport, ServingLoop, k_opt_linear,
                                           k_opt_quadratic, request_latency)


class OracleAdapter:
    def __init__(self, oracle_mod, dim, entries, items, policy=0):
        self.o = oracle_mod.OracleCache(dim=dim, entry_capacity=entries, latent_capacity=items)
        self.cap_e, self.cap_i, self.policy = entries, items, policy
        self.capacity_entries, self.capacity_items = entries, items

    def lookup(self, q):
        r = self.o.query(q, topk=1, want_latents=False, apply_counters=True)
        return r["ids"][:, 0], r["k"]

    def admit(self, emb, lat):
        rc, _, _ = self.o.insert(emb)
        assert rc == 0

    def evict(self, n):
        rc, ev, d = self.o.evict(n, policy=self.policy)
        assert rc == 0
        return ev, d

    def free(self):
        return self.cap_e - self.o.live_entries, self.cap_i - self.o.live_items


def test_latency_identity():
    """hit at K -> l_s + C (N-K)/N + l_r; miss -> l_s + C (SPEC acceptance #1)."""
    lat = LatencyParams(C=8.59, l_s=0.1, l_r=0.05, N=50)
    assert request_latency(25, lat) == 0.1 + 8.59 * 25 / 50 + 0.05
    assert request_latency(5, lat) == 0.1 + 8.59 * 45 / 50 + 0.05
    assert request_latency(0, lat) == 0.1 + 8.59


def test_savings_worked_example():
    """P:847 / SPEC S:521: h(25) = 0.08 at N = 50 contributes 0.04; all hits at K = 25 -> 0.5;
    overall hit-rate = sum h_opt ({.08,.1,.2,.47,.08} -> 0.93)."""
    r = RunReport(k_values=synth.K_VALUES, requests=100, hits_at={25: 8})
    assert r.f_c(50) == pytest.approx(0.04) and r.summary(LatencyParams())["per_k_savings"][25] == pytest.approx(0.04)
    assert RunReport(k_values=synth.K_VALUES, requests=10, hits_at={25: 10}).f_c(50) == 0.5
    r = RunReport(k_values=synth.K_VALUES, requests=100, hits_at={5: 8, 10: 10, 15: 20, 20: 47, 25: 8})
    assert r.hit_rate == pytest.approx(0.93)
    h = r.h()
    assert all(h[a] >= h[b] for a, b in zip(synth.K_VALUES, synth.K_VALUES[1:]))   # non-increasing
    assert h[5] == pytest.approx(r.hit_rate)


@pytest.mark.parametrize("K_T,N", [(50, 50), (30, 50), (40, 100)])
def test_footnote_closed_forms_vs_numeric_maximum(K_T, N):
    """maximise f_C(K) = h(K) K / N numerically on a fine grid and compare with the
    closed forms (linear: K_T/2, K_T/(4N); quadratic: K_T/sqrt(3), 2 K_T/(3 sqrt(3) N))."""
    K = np.linspace(0.0, K_T, 200001)
    for shape, fn in (("linear", k_opt_linear), ("quadratic", k_opt_quadratic)):
        h = 1 - K / K_T if shape == "linear" else 1 - (K / K_T) ** 2
        f = h * K / N
        i = int(np.argmax(f))
        k_opt, f_max = fn(K_T, N)
        assert abs(K[i] - k_opt) < 1e-3 and abs(f[i] - f_max) < 1e-9
    assert k_opt_quadratic(K_T, N)[1] > k_opt_linear(K_T, N)[1]      # "> K_T/4N"
    assert k_opt_linear(50, 50) == (25, 0.25)
    assert k_opt_quadratic(50, 50)[1] == pytest.approx(2 * 50 / (3 * math.sqrt(3) * 50))


def _stream(universe, cl, n_batches, b, seed):
    for i in range(n_batches):
        q, _, _ = synth.queries(universe, cl, b, seed=seed + i)
        yield q


def test_replay_accounting_and_determinism(oracle_mod):
    universe, cl = synth.entries(400, seed=11, dim=64)
    reps = []
    for _ in range(2):
        cache = OracleAdapter(oracle_mod, 64, entries=60, items=250)
        loop = ServingLoop(cache, synth.K_VALUES, LatencyParams())
        for q in _stream(universe, cl, 12, 32, seed=5):
            loop.step(q)
        s = loop.report.summary(loop.lat)
        reps.append(s)
        assert s["requests"] == 12 * 32
        assert s["f_c"] == pytest.approx(s["f_c_from_steps"], abs=1e-12)          # SPEC acceptance #2
        assert s["hit_rate"] == pytest.approx(sum(s["h_opt"].values()))
        assert s["evicted_items"] > 0 and s["admitted_prompts"] > 0               # capacity pressure
        assert cache.o.live_items <= 250 and cache.o.live_entries <= 60
        lat = loop.lat
        exp = [request_latency(k, lat) for k in np.repeat(0, 0)]
        assert len(loop.report.latencies) == s["requests"] and not exp
    assert reps[0] == reps[1]                                                       # SPEC acceptance #10
