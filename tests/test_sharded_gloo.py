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


# ---- the levels protocol of ShardedCache.evict (the distributed fused eviction) ----
def _bin0(k):
    k = np.asarray(k, dtype=np.uint64)
    out = np.empty(len(k), dtype=np.int64)
    small = k < 64
    out[small] = k[small].astype(np.int64)
    kb = k[~small]
    e = np.floor(np.log2(kb.astype(np.float64))).astype(np.int64)
    e = np.where((np.uint64(1) << e.astype(np.uint64)) > kb, e - 1, e)            # exact floor(log2)
    e = np.where((np.uint64(2) << e.astype(np.uint64)) <= kb, e + 1, e)
    m = ((kb >> (e - 6).astype(np.uint64)) & np.uint64(63)).astype(np.int64)
    out[~small] = 64 + (e - 6) * 64 + m
    return out


class _FakeLevelsCache:
    """Numpy stand-in of one rank's k_evict_select phases (level 0: 4,096 log bins; later
    levels: 12-bit digits of key - lo; the same pick on every rank); what is under test is
    ShardedCache.evict's orchestration: levels until done, histograms all-reduced by the
    process group, the ranks' lists merged into the global eviction order."""
    granularity = 0

    def __init__(self, keys):
        self.keys = np.sort(np.asarray(keys, dtype=np.uint64))

    @property
    def evict_units(self):
        return len(self.keys)

    def evict_sel_begin(self, n):
        self.n = n

    def evict_sel_level(self, level, hist):
        k = self.keys
        if level == 0:
            h = np.bincount(_bin0(k), minlength=4096)
        else:
            inr = k[(k >= np.uint64(self.lo)) & ((k - np.uint64(self.lo)) >> np.uint64(self.w) == 0)]
            h = np.bincount(((inr - np.uint64(self.lo)) >> np.uint64(self.shift)).astype(np.int64), minlength=4096)
        hist.copy_(torch.from_numpy(h.astype(np.int32)))

    def evict_sel_pick(self, level, hist):
        h = hist.numpy().astype(np.int64)
        target = self.n if level == 0 else self.rem
        cum = np.cumsum(h)
        b = int(np.searchsorted(cum, target))
        before = int(cum[b] - h[b])
        if level == 0:
            if b < 64:
                self.lo, self.w = b, 0
            else:
                e, m = (b - 64) // 64 + 6, (b - 64) % 64
                self.w, self.lo = e - 6, (64 + m) << (e - 6)
            self.rem = self.n - before
        else:
            self.lo += b << self.shift
            self.w = self.shift
            self.rem -= before
        done = int(h[b]) == self.rem or self.w == 0
        self.shift = self.w - min(12, self.w)
        return done

    def evict_sel_apply(self, cap, lists=True):
        T = self.lo + (1 << self.w) - 1
        self.last = self.keys[self.keys <= np.uint64(T)]
        self.keys = self.keys[self.keys > np.uint64(T)]
        return self.last & np.uint64((1 << 35) - 1), np.zeros(0, np.uint64)

    def last_evicted_keys(self):
        return self.last


def _levels_worker(rank, port, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        from paper_2312_04429_b200.sharded import ShardedCache, TorchComm
        rng = np.random.default_rng(11)
        # item keys score << 35 | id << 3 | j: a never-accessed bulk plus hot items
        ids = rng.permutation(50_000)[:20_000].astype(np.uint64)
        score = np.where(rng.random(20_000) < 0.8, 0, rng.integers(1, 3000, 20_000)).astype(np.uint64)
        keys_all = np.unique((score << np.uint64(35)) | (ids << np.uint64(3)) | rng.integers(0, 5, 20_000).astype(np.uint64))
        sc = object.__new__(ShardedCache)
        sc.comm, sc.push, sc.cache = TorchComm(device="cpu"), False, _FakeLevelsCache(keys_all[rank::WORLD])
        ok = True
        taken = 0
        for nsel in (1, 777, 5000, 9000):
            ev, _ = sc.evict(nsel)
            want = np.sort(keys_all)[taken:taken + nsel] & np.uint64((1 << 35) - 1)
            ok &= bool(np.array_equal(ev, want))
            taken += nsel
        ret[rank] = ok
    finally:
        dist.destroy_process_group()


def test_levels_protocol_gloo_world2():
    port = _free_port()
    ret = mp.Manager().dict()
    mp.spawn(_levels_worker, args=(port, ret), nprocs=WORLD, join=True)
    assert ret[0] is True and ret[1] is True, dict(ret)
