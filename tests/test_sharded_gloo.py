"""The multi-GPU (entry-sharded) protocol on CPU with gloo, world_size 2.

The CUDA kernels cannot run here, so the per-rank compute is played by test stand-ins built
on the oracle / numpy; what is under test is the product's collective protocol
(paper_2312_04429_b200.sharded.query_protocol / evict_protocol), the global-id placement
rule (rank r holds ids with id % world == r) and that a merge of per-shard top-k lists under
(score desc, id asc) reproduces the unsharded answer exactly -- including cross-shard ties.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shard_ids(n, rank, world):
    return np.arange(rank, n, world)


def _worker(rank, port, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        import oracle
        from paper_2312_04429_b200.sharded import TorchComm, evict_protocol, query_protocol
        comm = TorchComm(device="cpu")
        n, dim, topk = 301, 64, 3
        emb, cl = synth.entries(n, seed=77, dim=dim)
        emb[200] = emb[101]                  # exact duplicate across the two shards (ids 101 / 200)
        mine = _shard_ids(n, rank, WORLD)
        shard = oracle.OracleCache(dim=dim, entry_capacity=n)
        shard.insert(emb[mine])              # local oracle id i  <->  global id mine[i]
        q_all, _, _ = synth.queries(emb, cl, 2 * 8, seed=78)
        q_all[3] = emb[101]
        q_local = torch.from_numpy(q_all[rank * 8:(rank + 1) * 8])

        def local_fn(qg):
            r = shard.query(qg.numpy(), topk=topk, want_latents=False, apply_counters=False)
            gid = np.where(r["ids"] == oracle.NO_ID, -1, mine[np.minimum(r["ids"], len(mine) - 1).astype(np.int64)])
            return torch.from_numpy(np.stack([r["raw"], gid.astype(np.float64)], axis=-1))  # [b][topk][2]

        def merge_fn(b, row0, nb, recs_all):
            ra = recs_all.numpy()                # [world][b][topk][2]
            out = []
            for i in range(row0, row0 + nb):
                cand = [(ra[w, i, t, 0], int(ra[w, i, t, 1])) for w in range(WORLD) for t in range(topk)
                        if ra[w, i, t, 1] >= 0]
                cand.sort(key=lambda x: (-x[0], x[1]))
                out.append([c[1] for c in cand[:topk]])
            return out

        got = query_protocol(comm, q_local, topk, local_fn, merge_fn)
        full = oracle.OracleCache(dim=dim, entry_capacity=n)
        full.insert(emb)
        want = full.query(q_all[rank * 8:(rank + 1) * 8], topk=topk, want_latents=False, apply_counters=False)
        ok_query = all(list(map(int, want["ids"][i])) == got[i] for i in range(8))

        # distributed exact selection of the n lowest keys over the two shards
        rng = np.random.default_rng(5)
        keys_all = np.unique(rng.integers(0, 2 ** 40, size=4000, dtype=np.int64).astype(np.uint64))
        keys = keys_all[rank::WORLD]
        nsel = 777
        state = {"prefix": 0, "mask": 0, "remaining": nsel}
        hist = torch.zeros(256, dtype=torch.int64)

        def hist_fn(st, p, h):
            shift = 56 - 8 * p
            sel = keys[(keys & np.uint64(st["mask"])) == np.uint64(st["prefix"])]
            h.copy_(torch.from_numpy(np.bincount(((sel >> np.uint64(shift)) & np.uint64(255)).astype(np.int64),
                                                 minlength=256)))

        def pick_fn(h, st, p):
            shift, cum = 56 - 8 * p, 0
            for d in range(256):
                if cum + int(h[d]) >= st["remaining"]:
                    st["prefix"] |= d << shift
                    st["remaining"] -= cum
                    break
                cum += int(h[d])
            st["mask"] |= 255 << shift

        evict_protocol(comm, nsel, state, hist, hist_fn, pick_fn)
        local_sel = keys[keys <= np.uint64(state["prefix"])]
        counts = comm.all_gather(torch.tensor([len(local_sel)]))
        ok_evict = (int(state["prefix"]) == int(np.sort(keys_all)[nsel - 1]) and int(counts.sum()) == nsel)
        ret[rank] = (ok_query, ok_evict)
    finally:
        dist.destroy_process_group()


def test_sharded_protocol_gloo_world2():
    port = _free_port()
    ret = mp.Manager().dict()
    mp.spawn(_worker, args=(port, ret), nprocs=WORLD, join=True)
    assert ret[0] == (True, True) and ret[1] == (True, True), dict(ret)
