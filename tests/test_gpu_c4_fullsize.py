"""Parity at the default bench's full size and launch configuration (C4 at N = 1, BASELINE.json
configs[3]): a 10M-entry cache built exactly as bench.py builds it (on-device synthetic rows,
aliased latent pool, one-rank ShardedCache with the fused push exchange), one 16,384-query
batch, and 24 sampled rows checked against the fp64 oracle over ALL 10M entries.

The oracle cannot hold 10M x 768 fp64 rows at once, so it runs on ten 1M-entry slices of the
same rows (each slice its own plain oracle: normalise, exhaustive cosine, full sort) and the
global answer is the best of the slices' answers under the total order (score desc, id asc) --
the definition of a maximum over a partition, nothing more.  Accept rules as tests/parity.py
(strict tier 2^-12 on the top-1 gap, scores within 1e-4, K by Fig. 11 + holes on the oracle's
score, latent bytes exact against the aliased pool)."""
import numpy as np
import pytest
import torch

import synth
from tests.parity import TAU_SCORE, TAU_STRICT, _oracle_query_rows, hole_resolve

pytestmark = pytest.mark.gpu

N, B_GLOBAL, L, POOL = 10_000_000, 16_384, 4 * 64 * 64 * 2, 262_144
SLICE = 1_000_000
NO_ID = 0xFFFFFFFFFFFFFFFF


def test_c4_full_size_sampled_parity(oracle_mod):
    import socket
    import torch.distributed as dist
    from paper_2312_04429_b200 import binding as B, sharded as S
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("gloo", rank=0, world_size=1, init_method=f"tcp://127.0.0.1:{port}")
    try:
        # ---- the bench's C4 construction (bench.py: run_sharded) ----
        sc = S.ShardedCache(S.TorchComm(device="cpu"), entry_capacity=N + 1024, latent_capacity=POOL, dim=768,
                            latent_bytes=L, latent_alias=True, push_max_nb=B_GLOBAL, push_max_topk=1)
        for s0 in range(0, POOL, 8192):
            m = min(8192, POOL - s0)
            sc.cache.pool_write(s0, synth.latents_torch(s0, m, 1, L, seed=7, device="cuda").view(m, L))
        E = synth.TorchEntries(N, seed=1000, device="cuda")
        pres = synth.present_masks(N, seed=1000)
        for s0 in range(0, N, 65536):
            m = min(65536, N - s0)
            sc.insert(E.rows(torch.arange(s0, s0 + m, dtype=torch.int64, device="cuda")), None,
                      present=pres[s0:s0 + m])
        q, _, _ = E.queries(B_GLOBAL, qseed=1001)
        out = sc.alloc_outputs(B_GLOBAL, 1, latents=True)
        sc.query_into(q, out)
        torch.cuda.synchronize()
        sc.cache.push_status()
        rows = np.random.default_rng(4).choice(B_GLOBAL, 24, replace=False)
        gid = out["ids"][:, 0].cpu().numpy().view(np.uint64)[rows]
        gsc = out["scores"][:, 0].cpu().numpy()[rows]
        gk = out["k"].cpu().numpy()[rows]
        glat = out["latents"].cpu().numpy()[rows]
        qh = q.cpu().numpy()[rows]
    finally:
        dist.destroy_process_group()
    del sc
    torch.cuda.empty_cache()

    # ---- the oracle over ten 1M-entry slices: best of the slices' top-2 under (score desc, id asc) ----
    best = [[] for _ in rows]          # (score, -id) candidates per sampled row
    s_of_gpu = np.full(len(rows), np.nan)
    kmap = None
    for s0 in range(0, N, SLICE):
        x = E.rows(torch.arange(s0, s0 + SLICE, dtype=torch.int64, device="cuda")).cpu().numpy()
        o = oracle_mod.OracleCache(dim=768, entry_capacity=SLICE, latent_capacity=5 * SLICE)
        rc, ids, _ = o.insert(x, present=pres[s0:s0 + SLICE])
        assert rc == 0 and len(ids) == SLICE
        res = _oracle_query_rows(o, qh, range(len(rows)), 2)
        for i in range(len(rows)):
            for t in range(2):
                lid = int(res["ids"][i, t])
                if lid != NO_ID:
                    best[i].append((float(res["raw"][i, t]), -(lid + s0)))
            if s0 <= int(gid[i]) < s0 + SLICE:   # the fp64 score of the GPU's entry, from its slice
                s_of_gpu[i] = o.score_id(qh[i], int(gid[i]) - s0)
        kmap = o
        del o, x
    checked = exempt = 0
    for i in range(len(rows)):
        top = sorted(best[i], reverse=True)[:2]
        (s1, n1), (s2, _) = top[0], top[1]
        oid = -n1
        if s1 - s2 >= TAU_STRICT:
            assert int(gid[i]) == oid, f"row {rows[i]}: gpu {gid[i]} != oracle {oid} (gap {s1 - s2:.3g})"
        else:
            exempt += 1
            assert abs(s_of_gpu[i] - s1) <= TAU_STRICT, f"row {rows[i]}: gpu id outside the tau band"
        sg = s_of_gpu[i]
        assert abs(float(gsc[i]) - min(max(sg, -1.0), 1.0)) <= TAU_SCORE, (rows[i], gsc[i], sg)
        want = hole_resolve(kmap.select_k(sg), int(pres[int(gid[i])]), synth.K_VALUES)
        if int(gk[i]) != want:
            alt = {hole_resolve(kmap.select_k(sg + d), int(pres[int(gid[i])]), synth.K_VALUES)
                   for d in (-TAU_STRICT, TAU_STRICT)}
            assert int(gk[i]) in alt, (rows[i], gk[i], want)
        if gk[i] > 0:   # the aliased pool slot's stamped bytes
            j = synth.K_VALUES.index(int(gk[i]))
            slot = B.alias_slot(int(gid[i]), j, POOL)
            assert np.array_equal(glat[i], synth.latents_np(np.array([slot]), 1, L, seed=7)[0, 0]), rows[i]
        checked += 1
    assert checked == len(rows) and exempt <= 2
