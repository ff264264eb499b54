"""Eviction at C5's per-rank scale (100M entries over 8 GPUs -> 12.5M per rank):
LCBFU cache_evict of 1% of the live items after a few query batches, timed end to end (the
call is host-synchronous), then the re-insertion of as many fresh prompts as entries were
removed; EVICT_REPS rounds (default 3).
usage: [EVICT_REPS=n] python scripts/evict_scale.py [n_entries] [policy] [granularity] [alias]
(alias 0: a latent pool of 5 slots per entry, 256 B each, whose freed slots the eviction lists
-- as in the C2 bench cache; default 1: the aliased pool of C4/C5)"""
import json
import sys
import time

import numpy as np
import torch

import synth
from paper_2312_04429_b200 import binding as B


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 12_500_000
    policy = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    gran = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    alias = int(sys.argv[4]) if len(sys.argv) > 4 else 1
    D = 768
    g = B.NirvanaCache(entry_capacity=n + 1024, latent_capacity=(1 << 16) if alias else 5 * (n + 1024), dim=D,
                       latent_bytes=256, latent_alias=bool(alias), evict_granularity=gran)
    g.set_evict_policy(policy)
    if "EVICT_WINDOW" in __import__("os").environ:   # the single-sweep window's stride (-1 auto, 0 off)
        B.debug_evict_window(g, int(__import__("os").environ["EVICT_WINDOW"]))
    E = synth.TorchEntries(n, seed=5, device="cuda")
    pres = synth.present_masks(n, seed=5)
    t0 = time.perf_counter()
    for s in range(0, n, 65536):
        m = min(65536, n - s)
        g.insert(E.rows(torch.arange(s, s + m, dtype=torch.int64, device="cuda")), None, present=pres[s:s + m])
    torch.cuda.synchronize()
    t_ins = time.perf_counter() - t0
    for r in range(3):                       # give the counters some non-zero f
        q, _, _ = E.queries(16384, qseed=11 + r)
        g.query(q, topk=1, latents=False)
    torch.cuda.synchronize()
    res = dict(entries=n, policy=policy, granularity=gran, alias=alias, insert_s=t_ins, live_items=g.live_items)
    units = g.live_entries if gran else g.live_items
    for rep in range(int(__import__("os").environ.get("EVICT_REPS", "3"))):
        k = max(1, units // 100)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ev, dirty = g.evict(k, view=True)   # the lists in the library's pinned staging, no copy
        t = time.perf_counter() - t0
        # re-insert as many fresh prompts as entries were removed (the C5 round's second half)
        nn = len(dirty)
        rows = E.rows(torch.arange(n + 10_000_000 * (rep + 1), n + 10_000_000 * (rep + 1) + nn,
                                   dtype=torch.int64, device="cuda")) if nn else None
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        if nn:
            g.insert(rows, None)
        torch.cuda.synchronize()
        ti = time.perf_counter() - t1
        res[f"evict{rep}"] = dict(n=k, ms=1e3 * t, dirty=nn, insert_ms=1e3 * ti)
    # HBM bytes per pass: present + ids (4 + 4) + the policy's per-item column (5 x 4) per slot
    res["bytes_per_pass"] = (n + 1024) * (8 + 20)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
