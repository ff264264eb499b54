"""Sharding invariance on one GPU: P virtual ranks (separate caches, peer-pointer merge path)
must give results identical to one unsharded cache -- ids, scores (bitwise), K, latent bytes,
LCBFU counters, eviction sets -- and agree with the oracle."""
import numpy as np
import pytest
import torch

import synth
from tests.parity import check_batch, gpu_to_numpy

pytestmark = pytest.mark.gpu
L = 256


@pytest.fixture(scope="module")
def mods():
    from paper_2312_04429_b200 import binding, sharded
    return binding, sharded


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("topk", [1, 4])
def test_virtual_shards_equal_single_cache(mods, oracle_mod, world, topk):
    B, S = mods
    n = 1500
    emb, cl = synth.entries(n, seed=31 + world)
    emb[1400] = emb[7]                                     # cross-shard exact tie (ids 7 / 1400)
    pres = synth.present_masks(n, seed=31, hole_frac=0.2)
    lat = synth.latents_np(np.arange(n), 5, L, seed=31)
    single = B.NirvanaCache(entry_capacity=n, dim=768, latent_bytes=L)
    vs = S.VirtualShards(world, entry_capacity=n, dim=768, latent_bytes=L)
    et, lt = torch.from_numpy(emb).cuda(), torch.from_numpy(lat).cuda()
    ids1, _ = single.insert(et, lt, present=pres)
    ids2, _ = vs.insert(et, lt, present=pres)
    assert np.array_equal(ids1, ids2)
    o = oracle_mod.OracleCache(dim=768, entry_capacity=n, latent_bytes=L)
    o.insert(emb, latents=lat, present=pres)
    b = 48 * world
    for rnd in range(2):
        q, _, _ = synth.queries(emb, cl, b, seed=200 + rnd)
        q[5] = emb[7]
        qt = torch.from_numpy(q).cuda()
        a = gpu_to_numpy(single.query(qt, topk=topk))
        s = gpu_to_numpy(vs.query(qt, topk=topk))
        assert np.array_equal(a["ids"], s["ids"])
        assert np.array_equal(a["scores"].view(np.uint32), s["scores"].view(np.uint32))
        assert np.array_equal(a["k"], s["k"]) and np.array_equal(a["status"], s["status"])
        hit = a["k"] > 0
        assert np.array_equal(a["latents"][hit], s["latents"][hit])
        assert a["ids"][5, 0] == 7
        check_batch(s, o, q, topk, expected_latent=lambda e, k: lat[e, synth.K_VALUES.index(k)])
    for e in range(0, n, 7):
        assert np.array_equal(single.meta(e)[0], vs.meta(e)[0]) and single.meta(e)[1] == vs.meta(e)[1]
    # distributed eviction == single-cache eviction == oracle, in eviction order (keys are unique)
    for nev in (333, 1200):
        e1, d1 = single.evict(nev)
        e2, d2 = vs.evict(nev)
        rc, e3, d3 = o.evict(nev)
        assert np.array_equal(e1, e2) and np.array_equal(e3, e2)   # same order (the API contract)
        assert np.array_equal(d1, d2) and np.array_equal(d3, d2)
    q, _, _ = synth.queries(emb, cl, b, seed=300)
    qt = torch.from_numpy(q).cuda()
    a = gpu_to_numpy(single.query(qt, topk=topk))
    s = gpu_to_numpy(vs.query(qt, topk=topk))
    assert np.array_equal(a["ids"], s["ids"]) and np.array_equal(a["k"], s["k"])


def test_sharded_world1_evict_is_the_fused_eviction(oracle_mod):
    """A one-rank ShardedCache (bench C5 at N = 1) evicts through the fused single-launch path:
    the same lists as one cache and the oracle."""
    import socket
    import torch.distributed as dist
    from paper_2312_04429_b200 import binding as B, sharded as S
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("gloo", rank=0, world_size=1, init_method=f"tcp://127.0.0.1:{port}")
    try:
        n = 900
        emb, cl = synth.entries(n, seed=23)
        sc = S.ShardedCache(S.TorchComm(device="cpu"), entry_capacity=n, dim=768, latent_bytes=0,
                            push_max_nb=64, push_max_topk=1)
        single = B.NirvanaCache(entry_capacity=n, dim=768, latent_bytes=0)
        o = oracle_mod.OracleCache(dim=768, entry_capacity=n, latent_capacity=5 * n)
        for c in (sc, single):
            c.insert(torch.from_numpy(emb).cuda())
        o.insert(emb)
        q, _, _ = synth.queries(emb, cl, 64, seed=24)
        out = sc.alloc_outputs(64, 1, False)
        sc.query_into(torch.from_numpy(q).cuda(), out)
        single.query(torch.from_numpy(q).cuda(), latents=False)
        check_batch(gpu_to_numpy(out), o, q, 1)
        e1, d1 = sc.evict(700)
        e2, d2 = single.evict(700)
        rc, e3, d3 = o.evict(700)
        assert np.array_equal(e1, e2) and np.array_equal(e1, e3) and np.array_equal(d1, d2) and np.array_equal(d1, d3)
        assert sc.evict(10, lists=False) == (10, len(single.evict(10)[1]))
    finally:
        dist.destroy_process_group()


def _proc_nccl_path(rank, port, ret):
    """One rank of the all-gather (non-push) path: queries and records all-gathered by the
    process group, the fused eviction's level histograms all-reduced by it."""
    import os
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        torch.cuda.set_device(0)
        from paper_2312_04429_b200 import binding as B, sharded as S
        n, bl = 800, 32
        emb, cl = synth.entries(n, seed=57)
        sc = S.ShardedCache(S.TorchComm(device="cpu"), entry_capacity=n, dim=768, latent_bytes=0)
        sc.insert(torch.from_numpy(emb).cuda())
        single = B.NirvanaCache(entry_capacity=n, dim=768, latent_bytes=0)
        single.insert(torch.from_numpy(emb).cuda())
        ok = True
        for rnd in range(2):
            q, _, _ = synth.queries(emb, cl, 2 * bl, seed=58 + rnd)
            out = sc.alloc_outputs(bl, 1, False)
            sc.query_into(torch.from_numpy(q[rank * bl:(rank + 1) * bl]).cuda(), out)
            full = single.query(torch.from_numpy(q).cuda(), latents=False)
            ok &= bool(torch.equal(out["ids"], full["ids"][rank * bl:(rank + 1) * bl]))
            e1, d1 = sc.evict(150)
            e2, d2 = single.evict(150)
            ok &= bool(np.array_equal(e1, e2) and np.array_equal(d1, d2))
        ret[rank] = ok
    except Exception as e:   # noqa: BLE001
        ret[rank] = repr(e)
    finally:
        dist.destroy_process_group()


def test_two_processes_allgather_path_levels_eviction():
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    ret = mgr.dict()
    procs = [ctx.Process(target=_proc_nccl_path, args=(r, port, ret)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    for p in procs:
        if p.is_alive():
            p.kill()
    assert dict(ret) == {0: True, 1: True}, dict(ret)
