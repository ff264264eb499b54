"""Oracle of the NEXT-1 serving loop -- TEST INFRASTRUCTURE (only tests/ may import it).

A second, plain implementation of what the product's paper_2312_04429_b200/serving.py does
around the lookup, written from the paper and sharing no code with it:

  * per request (Alg. 1): K = the lookup's resolved step (0 = no match / no
    suitable state -> scratch); latency l_s + C (N - K)/N + l_r on a hit (Eq. latency,
    P:297-300), l_s + C on a miss;
  * savings: f_C = sum_K h_opt(K) K / N (Eq. compute_saving), h_opt(K) = the
    fraction of requests served at exactly K, overall hit-rate = sum_K h_opt(K);
  * admission (LCBFU insertion): every miss inserts its prompt embedding and all
    |K| intermediate states; inserts go without eviction until the storage limit, after
    which every insertion is preceded by an eviction of the policy's lowest-scored items.
    Reading R26: a batch's misses are admitted together after ONE eviction of the
    batch's shortfall -- the items missing for all of them, or |K| items per entry slot
    missing (entries come back only when all their states are gone) -- capped at the live
    items; misses that still do not fit are not admitted (in request order).

The cache is the fp64 oracle (oracle.OracleCache); the K of each request comes from the
caller (the parity harness validates the GPU's K against this oracle request by request and
hands the accepted value in, so both loops see the same decisions on near-ties).
"""
from __future__ import annotations

import numpy as np


class OracleServing:
    def __init__(self, orc, k_values, entry_capacity, item_capacity, policy=0, C=8.59, l_s=0.1, l_r=0.05, N=50):
        self.orc = orc
        self.k_values = list(k_values)
        self.entry_capacity, self.item_capacity, self.policy = entry_capacity, item_capacity, policy
        self.C, self.l_s, self.l_r, self.N = C, l_s, l_r, N
        self.requests = 0
        self.served_at = {k: 0 for k in self.k_values}   # requests served at exactly K
        self.latencies = []
        self.log = []

    def latency(self, K):
        if K > 0:
            return self.l_s + self.C * (self.N - K) / self.N + self.l_r
        return self.l_s + self.C

    def step(self, q, k_used):
        lat = []
        misses = []
        for i in range(len(k_used)):
            K = int(k_used[i])
            self.requests += 1
            if K > 0:
                self.served_at[K] += 1
            else:
                misses.append(i)
            lat.append(self.latency(K))
        self.latencies.extend(lat)
        # LCBFU admission (reading R26)
        nk = len(self.k_values)
        free_items = self.item_capacity - self.orc.live_items
        free_entries = self.entry_capacity - self.orc.live_entries
        n_evict = 0
        if len(misses) * nk > free_items:
            n_evict = len(misses) * nk - free_items
        if len(misses) > free_entries:
            n_evict = max(n_evict, (len(misses) - free_entries) * nk)
        n_evict = min(n_evict, self.orc.live_items)
        evicted = dirty = np.zeros(0, np.uint64)
        if n_evict > 0:
            rc, evicted, dirty = self.orc.evict(n_evict, policy=self.policy)
            assert rc == 0
        free_items = self.item_capacity - self.orc.live_items
        free_entries = self.entry_capacity - self.orc.live_entries
        admit = min(len(misses), free_entries, free_items // nk)
        if admit > 0:
            rc, _, _ = self.orc.insert(np.asarray(q)[misses[:admit]])
            assert rc == 0
        self.log.append(dict(k=np.asarray(k_used, np.int32).copy(), latency=lat, evicted=evicted, dirty=dirty,
                             admitted=max(admit, 0)))

    def h_opt(self):
        return {k: self.served_at[k] / max(1, self.requests) for k in self.k_values}

    def f_c(self):
        return sum(h * k for k, h in self.h_opt().items()) / self.N

    def hit_rate(self):
        return sum(self.h_opt().values())
