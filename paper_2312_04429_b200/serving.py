"""Alg. 1 serving loop over a request stream + the paper's analytic accounting.

Per batch of prompt embeddings (batched):
  lookup      cache_query_batch -> K_used per request (0 = generate from scratch)
  hit         the diffusion model runs N - K_used steps from the retrieved state
  miss        it runs all N steps; LCBFU insertion then admits the prompt's embedding and
              all |K| intermediate states, evicting the policy's lowest-scored
              items first when the cache is full ("every insertion is preceded by an
              eviction")
Accounting:
  latency     hit  l_s + C (N - K)/N + l_r   (Eq. eq:latency)
              miss l_s + C
  f_C         sum_K hits(K) K / (requests N)  (Eq. eq:compute_saving, per K h(K) K/N)
  h_opt(K)    fraction of requests served at exactly K; h(K) = sum_{K' >= K} h_opt(K');
              overall hit-rate h(min K) = sum_K h_opt(K) (Eq. eq:overall_hit)
The loop only orchestrates library calls; every lookup, eviction and insertion runs in the
CUDA library through the cache object it is given.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass
class LatencyParams:
    """Paper constants: C ~ 8.59 s for N = 50 DDIM steps on an A10g, l_s of
    the order of 100 ms; l_r is not given numerically (SPEC's default 50 ms)."""
    C: float = 8.59
    l_s: float = 0.1
    l_r: float = 0.05
    N: int = 50


@dataclass
class RunReport:
    k_values: tuple
    requests: int = 0
    hits_at: dict = field(default_factory=dict)      # K -> count
    latencies: list = field(default_factory=list)
    steps: int = 0
    evicted_items: int = 0
    admitted_prompts: int = 0
    dirty_removed: int = 0

    def h_opt(self):
        return {k: self.hits_at.get(k, 0) / max(1, self.requests) for k in self.k_values}

    def h(self):
        ho = self.h_opt()
        return {k: sum(v for kk, v in ho.items() if kk >= k) for k in self.k_values}

    @property
    def hit_rate(self):
        return sum(self.h_opt().values())

    def f_c(self, N):
        return sum(k * c for k, c in self.hits_at.items()) / (max(1, self.requests) * N)

    def summary(self, lat: LatencyParams):
        L = np.asarray(self.latencies)
        return dict(requests=self.requests, hit_rate=self.hit_rate, h_opt=self.h_opt(), h=self.h(),
                    f_c=self.f_c(lat.N), f_c_from_steps=1.0 - self.steps / (max(1, self.requests) * lat.N),
                    per_k_savings={k: v * k / lat.N for k, v in self.h_opt().items()},
                    mean_latency_s=float(L.mean()) if len(L) else 0.0,
                    p50_latency_s=float(np.percentile(L, 50)) if len(L) else 0.0,
                    p99_latency_s=float(np.percentile(L, 99)) if len(L) else 0.0,
                    latency_reduction_vs_scratch=1.0 - float(L.mean()) / (lat.C) if len(L) else 0.0,
                    evicted_items=self.evicted_items, admitted_prompts=self.admitted_prompts,
                    dirty_removed=self.dirty_removed)


def request_latency(k_used: int, lat: LatencyParams) -> float:
    """Eq. eq:latency for a hit at K; l_s + C for a miss."""
    if k_used > 0:
        return lat.l_s + lat.C * (lat.N - k_used) / lat.N + lat.l_r
    return lat.l_s + lat.C


class ServingLoop:
    """cache: an object with lookup(q) -> (ids, K), admit(emb, latents), evict(n) -> (evicted,
    dirty), free() -> (free entries, free items), capacity_items and, with use_predictor,
    train_predictor(), predict(q) -> bool flags and (optional) peek(q) -> K without counting
    an access; see GpuCache for the library adapter.

    With the match predictor (Alg. 1 line 2) a predicted miss goes straight
    to scratch generation WITHOUT the search (latency C, arrow 1 of the overview): only
    the rows the predictor accepts are looked up, so rejected requests count no access.  It is
    retrained when more than 5% of the cached entries changed since the last training
    (P:485-486).  Whether a rejected request would have hit (recall) is measured
    with the cache's read-only peek, which leaves the eviction state untouched.

    keep_log: record every step (per-request K and latency, evicted / dirty ids, admitted
    prompts) in self.log -- the per-request parity tests compare it with the oracle's loop."""

    def __init__(self, cache, k_values, lat: LatencyParams = LatencyParams(), make_latents=None,
                 use_predictor: bool = False, retrain_threshold: float = 0.05, keep_log: bool = False):
        self.cache, self.k_values, self.lat = cache, tuple(k_values), lat
        self.make_latents = make_latents
        self.report = RunReport(k_values=self.k_values)
        self._admitted = 0
        self.use_predictor, self.retrain_threshold = use_predictor, retrain_threshold
        self._changed = 0          # entries admitted + removed since the last training
        self._trained_on = 0
        self.pred_stats = dict(predicted_true=0, predicted_true_hit=0, predicted_false=0,
                               predicted_false_would_hit=0, searched_missed=0, retrains=0)
        self.keep_log, self.log = keep_log, []

    def _maybe_retrain(self):
        fe, _ = self.cache.free()
        live = self.cache.capacity_entries - fe
        if live <= 0:
            return False
        if self._trained_on == 0 or self._changed > self.retrain_threshold * max(1, self._trained_on):
            self.cache.train_predictor()
            self._trained_on, self._changed = live, 0
            self.pred_stats["retrains"] += 1
        return True

    def step(self, q: np.ndarray):
        b = len(q)
        gate = None
        if self.use_predictor and self._maybe_retrain():
            gate = np.asarray(self.cache.predict(q), dtype=bool)
        ids = np.full(b, np.iinfo(np.uint64).max, dtype=np.uint64)
        ks = np.zeros(b, dtype=np.int32)
        searched = np.arange(b) if gate is None else np.nonzero(gate)[0]
        if len(searched):   # Alg. 1 lines 4-5: search_VDB + heuristics_K for the accepted rows only
            ids_s, ks_s = self.cache.lookup(q[searched] if gate is not None else q)
            ids[searched], ks[searched] = ids_s, ks_s
        r = self.report
        lat_step = []
        if gate is not None:
            ps = self.pred_stats
            rej = np.nonzero(~gate)[0]
            ps["predicted_true"] += len(searched)
            ps["predicted_true_hit"] += int(np.count_nonzero(ks[searched] > 0))
            ps["searched_missed"] += int(np.count_nonzero(ks[searched] == 0))
            ps["predicted_false"] += len(rej)
            if len(rej) and hasattr(self.cache, "peek"):   # would-hit, without counting an access
                ps["predicted_false_would_hit"] += int(np.count_nonzero(self.cache.peek(q[rej]) > 0))
        for i in range(b):
            k = int(ks[i])
            r.requests += 1
            if k > 0:
                r.hits_at[k] = r.hits_at.get(k, 0) + 1
            r.steps += self.lat.N - k
            # a predicted miss skips the search: scratch generation alone, latency C (arrow 1)
            lt = request_latency(k, self.lat) if gate is None or gate[i] else self.lat.C
            r.latencies.append(lt)
            lat_step.append(lt)
        miss = np.nonzero(ks == 0)[0]
        ev = dirty = np.zeros(0, np.uint64)
        m = 0
        if len(miss):
            ev, dirty, m = self._admit(q[miss])
        if self.keep_log:
            self.log.append(dict(k=ks.copy(), latency=lat_step, evicted=np.asarray(ev, np.uint64),
                                 dirty=np.asarray(dirty, np.uint64), admitted=m))
        return ids, ks

    def predictor_summary(self):
        ps = dict(self.pred_stats)
        n = max(1, self.report.requests)
        ps["precision_c_p"] = ps["predicted_true_hit"] / max(1, ps["predicted_true"])
        ps["recall"] = ps["predicted_true_hit"] / max(1, ps["predicted_true_hit"] + ps["predicted_false_would_hit"])
        ps["wasted_search_fraction"] = ps["searched_missed"] / n
        return ps

    def _admit(self, emb: np.ndarray):
        """LCBFU admission of a batch's misses (reading R26): one eviction of the
        shortfall (items, or |K| items per missing entry slot; never more than the live items)
        before inserting; the misses that still do not fit are not admitted."""
        nk = len(self.k_values)
        need_e, need_i = len(emb), len(emb) * nk
        fe, fi = self.cache.free()
        short = max(0, need_i - fi)
        if fe < need_e:          # entries only come back when all of an entry's K are evicted
            short = max(short, (need_e - fe) * nk)
        short = min(short, self.cache.capacity_items - fi)   # the live items
        ev = dirty = np.zeros(0, np.uint64)
        if short > 0:
            ev, dirty = self.cache.evict(short)
            self.report.evicted_items += len(ev)
            self.report.dirty_removed += len(dirty)
            self._changed += len(dirty)
            fe, fi = self.cache.free()
        m = min(len(emb), fe, fi // nk)
        if m <= 0:
            return ev, dirty, 0
        lat = self.make_latents(self._admitted, m) if self.make_latents else None
        self.cache.admit(emb[:m], lat)
        self._admitted += m
        self._changed += m
        self.report.admitted_prompts += m
        return ev, dirty, m


class GpuCache:
    """ServingLoop adapter over binding.NirvanaCache (device buffers, CUDA library calls)."""

    def __init__(self, cache, device="cuda", nu: float = 0.001):
        import torch
        self.c, self.torch, self.device, self.nu = cache, torch, device, nu
        self.capacity_entries = cache.cfg.entry_capacity
        self.capacity_items = cache.cfg.latent_capacity
        self.last_out = None   # the last lookup's device outputs (ids, scores, k, ...)

    def train_predictor(self):
        self.c.train_predictor(nu=self.nu)

    def predict(self, q):
        flags, _ = self.c.predict(self.torch.from_numpy(np.ascontiguousarray(q)).to(self.device))
        return flags.cpu().numpy().astype(bool)

    def lookup(self, q):
        out = self.c.query(self.torch.from_numpy(np.ascontiguousarray(q)).to(self.device), topk=1)
        self.last_out = out
        return out["ids"][:, 0].cpu().numpy().view(np.uint64), out["k"].cpu().numpy()

    def peek(self, q):
        out = self.c.peek(self.torch.from_numpy(np.ascontiguousarray(q)).to(self.device), topk=1)
        return out["k"].cpu().numpy()

    def admit(self, emb, latents):
        self.c.insert(self.torch.from_numpy(np.ascontiguousarray(emb)).to(self.device), latents)

    def evict(self, n):
        return self.c.evict(n)

    def free(self):
        s = self.c.stats()
        return s["free_entries"], s["free_items"]


# ------------------------- footnote closed forms ------------------------------
def k_opt_linear(K_T: float, N: float):
    """h(K) = 1 - K/K_T  =>  f_C(K) = h(K) K/N is maximal at K_OPT = K_T/2 with
    f_C^max = K_T/(4N)."""
    return K_T / 2.0, K_T / (4.0 * N)


def k_opt_quadratic(K_T: float, N: float):
    """h(K) = 1 - (K/K_T)^2  =>  K_OPT = K_T/sqrt(3), f_C^max = 2 K_T/(3 sqrt(3) N)."""
    return K_T / math.sqrt(3.0), 2.0 * K_T / (3.0 * math.sqrt(3.0) * N)
