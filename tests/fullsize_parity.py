"""Sampled parity at a sharded config's FULL size, in the launch configuration bench.py times
(test infrastructure).  Used by tests/test_gpu_c4_fullsize.py (C4, every GPU run) and runnable
on its own for C5 (100M entries; ~30 min of oracle work on the box's host cores):

    python -m tests.fullsize_parity c5 [samples]

The cache is built exactly as bench.py's run_sharded builds it (on-device synthetic rows,
aliased latent pool, a one-rank ShardedCache with the fused push exchange), one query batch of
the bench's size runs, and `samples` rows are checked against the fp64 oracle over ALL entries.
The oracle cannot hold 10M-100M fp64 rows at once, so it runs on 1M-entry slices of the same
rows (each slice its own plain oracle: normalise, exhaustive cosine, full sort) and the global
answer is the best of the slices' answers under the total order (score desc, id asc) -- the
definition of a maximum over a partition, nothing more.  Accept rules as tests/parity.py
(strict tier 2^-12 on the top-1 gap, scores within 1e-4, K by Fig. 11 + holes on the oracle's
score, latent bytes exact against the aliased pool)."""
from __future__ import annotations

import json
import sys
import time

import numpy as np

NO_ID = 0xFFFFFFFFFFFFFFFF
L = 4 * 64 * 64 * 2
SLICE = 1_000_000
CONFIGS = {"c4": dict(n=10_000_000, b=16_384, pool=262_144, headroom=False),
           "c5": dict(n=100_000_000, b=16_384, pool=131_072, headroom=True)}


def run(oracle_mod, config: str = "c4", samples: int = 24, seed: int = 4) -> dict:
    import socket

    import torch
    import torch.distributed as dist

    import synth
    from paper_2312_04429_b200 import binding as B, sharded as S
    from tests.parity import TAU_SCORE, TAU_STRICT, _oracle_query_rows, hole_resolve

    cfg = CONFIGS[config]
    N, BG, POOL = cfg["n"], cfg["b"], cfg["pool"]
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    t0 = time.time()
    dist.init_process_group("gloo", rank=0, world_size=1, init_method=f"tcp://127.0.0.1:{port}")
    try:
        cap = N + (N // 200 if cfg["headroom"] else 0) + 1024
        sc = S.ShardedCache(S.TorchComm(device="cpu"), entry_capacity=cap, latent_capacity=POOL, dim=768,
                            latent_bytes=L, latent_alias=True, push_max_nb=BG, push_max_topk=1)
        for s0 in range(0, POOL, 8192):
            m = min(8192, POOL - s0)
            sc.cache.pool_write(s0, synth.latents_torch(s0, m, 1, L, seed=7, device="cuda").view(m, L))
        E = synth.TorchEntries(N, seed=1000, device="cuda")
        pres = synth.present_masks(N, seed=1000)
        for s0 in range(0, N, 65536):
            m = min(65536, N - s0)
            sc.insert(E.rows(torch.arange(s0, s0 + m, dtype=torch.int64, device="cuda")), None,
                      present=pres[s0:s0 + m])
        q, _, _ = E.queries(BG, qseed=1001)
        out = sc.alloc_outputs(BG, 1, latents=True)
        sc.query_into(q, out)
        torch.cuda.synchronize()
        sc.cache.push_status()
        rows = np.random.default_rng(seed).choice(BG, samples, replace=False)
        gid = out["ids"][:, 0].cpu().numpy().view(np.uint64)[rows]
        gsc = out["scores"][:, 0].cpu().numpy()[rows]
        gk = out["k"].cpu().numpy()[rows]
        glat = out["latents"].cpu().numpy()[rows]
        qh = q.cpu().numpy()[rows]
    finally:
        dist.destroy_process_group()
    del sc, out
    torch.cuda.empty_cache()
    t_gpu = time.time() - t0

    best = [[] for _ in rows]          # (score, -id) candidates per sampled row
    s_of_gpu = np.full(len(rows), np.nan)
    kmap = None
    for s0 in range(0, N, SLICE):
        x = E.rows(torch.arange(s0, min(N, s0 + SLICE), dtype=torch.int64, device="cuda")).cpu().numpy()
        o = oracle_mod.OracleCache(dim=768, entry_capacity=len(x), latent_capacity=5 * len(x))
        rc, ids, _ = o.insert(x, present=pres[s0:s0 + len(x)])
        assert rc == 0 and len(ids) == len(x)
        res = _oracle_query_rows(o, qh, range(len(rows)), 2)
        for i in range(len(rows)):
            for t in range(2):
                lid = int(res["ids"][i, t])
                if lid != NO_ID:
                    best[i].append((float(res["raw"][i, t]), -(lid + s0)))
            if s0 <= int(gid[i]) < s0 + len(x):   # the fp64 score of the GPU's entry, from its slice
                s_of_gpu[i] = o.score_id(qh[i], int(gid[i]) - s0)
        kmap = o
        del o, x
    rep = dict(config=config, entries=N, batch=BG, samples=int(len(rows)), exempt=0, hits=0, max_dscore=0.0)
    for i in range(len(rows)):
        top = sorted(best[i], reverse=True)[:2]
        (s1, n1), (s2, _) = top[0], top[1]
        oid = -n1
        if s1 - s2 >= TAU_STRICT:
            assert int(gid[i]) == oid, f"row {rows[i]}: gpu {gid[i]} != oracle {oid} (gap {s1 - s2:.3g})"
        else:
            rep["exempt"] += 1
            assert abs(s_of_gpu[i] - s1) <= TAU_STRICT, f"row {rows[i]}: gpu id outside the tau band"
        sg = s_of_gpu[i]
        d = abs(float(gsc[i]) - min(max(sg, -1.0), 1.0))
        rep["max_dscore"] = max(rep["max_dscore"], d)
        assert d <= TAU_SCORE, (rows[i], gsc[i], sg)
        mask = int(pres[int(gid[i])])
        want = hole_resolve(kmap.select_k(sg), mask, synth.K_VALUES)
        if int(gk[i]) != want:
            alt = {hole_resolve(kmap.select_k(sg + dd), mask, synth.K_VALUES) for dd in (-TAU_STRICT, TAU_STRICT)}
            assert int(gk[i]) in alt, (rows[i], gk[i], want)
        if gk[i] > 0:   # the aliased pool slot's stamped bytes
            rep["hits"] += 1
            j = synth.K_VALUES.index(int(gk[i]))
            slot = B.alias_slot(int(gid[i]), j, POOL)
            assert np.array_equal(glat[i], synth.latents_np(np.array([slot]), 1, L, seed=7)[0, 0]), rows[i]
    rep["gpu_s"] = round(t_gpu, 1)
    rep["total_s"] = round(time.time() - t0, 1)
    return rep


if __name__ == "__main__":
    import oracle
    oracle.build()
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
    ns = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    print(json.dumps(run(oracle, cfg, ns)), flush=True)
