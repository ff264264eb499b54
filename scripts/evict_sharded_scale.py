"""The distributed eviction with virtual ranks on one GPU (the same kernels and level protocol as
ShardedCache, collectives replaced by copies): P shards of n_per entries, LCBFU eviction of 1% of
the live items, single-sweep window on (auto) vs off, host wall per eviction.  Virtual ranks run
one after another, so a call costs ~P x one rank's time.
usage: python scripts/evict_sharded_scale.py [n_per] [P] [push]"""
import json
import sys
import time

import torch

import synth
from paper_2312_04429_b200 import binding as B, sharded as S


def main():
    n_per = int(sys.argv[1]) if len(sys.argv) > 1 else 6_250_000
    P = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    push = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    n = n_per * P
    vs = S.VirtualShards(P, entry_capacity=n_per + 4096, latent_capacity=1 << 16, dim=768, latent_bytes=256,
                         latent_alias=True, push_max_nb=(16384 // P if push else 0), push_max_topk=1)
    E = synth.TorchEntries(n, seed=7, device="cuda")
    pres = synth.present_masks(n, seed=7)
    for s0 in range(0, n, 65536):
        m = min(65536, n - s0)
        vs.insert(E.rows(torch.arange(s0, s0 + m, dtype=torch.int64, device="cuda")), None, present=pres[s0:s0 + m])
    for r in range(2):
        q, _, _ = E.queries(16384, qseed=21 + r)
        vs.query(q, latents=False)
    torch.cuda.synchronize()
    res = dict(n_per=n_per, P=P, push=push)
    for label, stride in (("window", -1), ("two_sweep", 0), ("window_again", -1)):
        for c in vs.caches:
            B.debug_evict_window(c, stride)
        ms = []
        for rep in range(3):
            live = sum(c.live_items for c in vs.caches)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ev, dirty = vs.evict(max(1, live // 100))
            torch.cuda.synchronize()
            ms.append(1e3 * (time.perf_counter() - t0))
            wins = [B.debug_evict_window(c) for c in vs.caches]
        res[label] = dict(ms=ms, windows=wins)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
