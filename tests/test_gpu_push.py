"""The fused push exchange (cache_push_*): queries stored into every rank's arena by the ingest
kernel, records stored into their owner's inbox by the local-merge kernel, epoch flags with
release/acquire at system scope -- no collective library on the data path.

* virtual ranks (one process, one stream, phase by phase): results identical to one
  unsharded cache over several batches (arena reuse), counters and eviction included;
* two PROCESSES sharing the GPU: the same through CUDA IPC mappings of each other's arenas,
  with the processes' own streams (gloo only carries the descriptors)."""
import os
import socket

import numpy as np
import pytest
import torch

import synth
from tests.parity import check_batch, gpu_to_numpy

pytestmark = pytest.mark.gpu
L = 256


@pytest.mark.parametrize("world,topk", [(2, 1), (3, 4), (4, 1), (4, 16)])
def test_push_virtual_shards_equal_single_cache(oracle_mod, world, topk):
    from paper_2312_04429_b200 import binding as B, sharded as S
    n = 1300
    emb, cl = synth.entries(n, seed=41 + world)
    emb[1200] = emb[9]                                      # cross-shard exact tie
    pres = synth.present_masks(n, seed=41, hole_frac=0.2)
    lat = synth.latents_np(np.arange(n), 5, L, seed=41)
    single = B.NirvanaCache(entry_capacity=n, dim=768, latent_bytes=L)
    bl = 40
    vs = S.VirtualShards(world, entry_capacity=n, dim=768, latent_bytes=L, push_max_nb=64, push_max_topk=16)
    et, lt = torch.from_numpy(emb).cuda(), torch.from_numpy(lat).cuda()
    single.insert(et, lt, present=pres)
    vs.insert(et, lt, present=pres)
    o = oracle_mod.OracleCache(dim=768, entry_capacity=n, latent_bytes=L)
    o.insert(emb, latents=lat, present=pres)
    for rnd in range(3):                                    # epochs 1..3 reuse the arenas
        q, _, _ = synth.queries(emb, cl, bl * world, seed=300 + rnd)
        q[3] = emb[9]
        qt = torch.from_numpy(q).cuda()
        a = gpu_to_numpy(single.query(qt, topk=topk))
        s = gpu_to_numpy(vs.query(qt, topk=topk))
        assert np.array_equal(a["ids"], s["ids"])
        assert np.array_equal(a["scores"].view(np.uint32), s["scores"].view(np.uint32))
        assert np.array_equal(a["k"], s["k"]) and np.array_equal(a["status"], s["status"])
        hit = a["k"] > 0
        assert np.array_equal(a["latents"][hit], s["latents"][hit])
        assert a["ids"][3, 0] == 9
        check_batch(s, o, q, topk, expected_latent=lambda e, k: lat[e, synth.K_VALUES.index(k)])
    for e in range(0, n, 11):
        assert np.array_equal(single.meta(e)[0], vs.meta(e)[0])
    for nev in (500, 77, 1200):                              # fused eviction: successive epochs
        e1, d1 = single.evict(nev)
        e2, d2 = vs.evict(nev)
        assert np.array_equal(e1, e2) and np.array_equal(d1, d2)   # global eviction order
        assert vs.stats()["live_items"] == single.live_items


def test_push_smaller_batch_and_bad_calls():
    """nb below the reserved maximum, a zero-row batch, and call-order errors."""
    from paper_2312_04429_b200 import binding as B, sharded as S
    n = 500
    emb, cl = synth.entries(n, seed=5)
    single = B.NirvanaCache(entry_capacity=n, dim=768, latent_bytes=0)
    vs = S.VirtualShards(2, entry_capacity=n, dim=768, latent_bytes=0, push_max_nb=300, push_max_topk=4)
    single.insert(torch.from_numpy(emb).cuda())
    vs.insert(torch.from_numpy(emb).cuda())
    for b in (2, 34, 0, 600):
        q, _, _ = synth.queries(emb, cl, max(b, 2), seed=b)
        qt = torch.from_numpy(q[:b]).cuda()
        a = gpu_to_numpy(single.query(qt, topk=4, latents=False)) if b else None
        s = gpu_to_numpy(vs.query(qt, topk=4, latents=False))
        if b:
            assert np.array_equal(a["ids"], s["ids"]) and np.array_equal(a["k"], s["k"])
    c = vs.caches[0]
    with pytest.raises(B.CacheError):
        c.push_scan(1, 1)                                   # before push_queries
    with pytest.raises(B.CacheError):
        c.push_queries(torch.zeros((301, 768), device="cuda"))   # nb > reserved maximum
    plain = B.NirvanaCache(entry_capacity=10, dim=768, latent_bytes=0)
    with pytest.raises(B.CacheError):
        plain.push_queries(torch.zeros((1, 768), device="cuda"))  # no arenas attached


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _proc(rank, port, world, ret):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2312_04429_b200 import binding as B, sharded as S
        n, bl = 900, 24
        emb, cl = synth.entries(n, seed=17)
        lat = synth.latents_np(np.arange(n), 5, L, seed=17)
        comm = S.TorchComm(device="cpu")
        sc = S.ShardedCache(comm, entry_capacity=n, dim=768, latent_bytes=L, push_max_nb=bl, push_max_topk=4)
        sc.insert(torch.from_numpy(emb).cuda(), torch.from_numpy(lat).cuda())
        single = B.NirvanaCache(entry_capacity=n, dim=768, latent_bytes=L)
        single.insert(torch.from_numpy(emb).cuda(), torch.from_numpy(lat).cuda())
        ok = True
        for rnd in range(3):
            q, _, _ = synth.queries(emb, cl, bl * world, seed=70 + rnd)
            mine = torch.from_numpy(q[rank * bl:(rank + 1) * bl]).cuda()
            out = sc.alloc_outputs(bl, 4, True)
            sc.query_into(mine, out, topk=4)
            torch.cuda.synchronize()
            full = gpu_to_numpy(single.query(torch.from_numpy(q).cuda(), topk=4))   # the whole global batch
            got = gpu_to_numpy(out)
            exp = {k: (v[rank * bl:(rank + 1) * bl] if v is not None else None) for k, v in full.items()}
            hit = exp["k"] > 0
            ok &= bool(np.array_equal(got["ids"], exp["ids"]) and np.array_equal(got["k"], exp["k"])
                       and np.array_equal(got["scores"].view(np.uint32), exp["scores"].view(np.uint32))
                       and np.array_equal(got["latents"][hit], exp["latents"][hit]))
        # the fused eviction across the two processes equals the reference cache's eviction (it
        # saw the same global batches, so its access counters are the sharded ones)
        for nev in (150, 600):
            ev, dirty = sc.evict(nev)
            e1, d1 = single.evict(nev)
            ok &= bool(np.array_equal(ev, e1) and np.array_equal(dirty, d1))
        ret[rank] = ok
    except Exception as e:                                   # noqa: BLE001
        ret[rank] = repr(e)
    finally:
        dist.destroy_process_group()


def test_push_two_processes_one_gpu():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    world, port = 2, _free_port()
    mgr = ctx.Manager()
    ret = mgr.dict()
    procs = [ctx.Process(target=_proc, args=(r, port, world, ret)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    for p in procs:
        if p.is_alive():
            p.kill()
    assert dict(ret) == {0: True, 1: True}, dict(ret)


@pytest.mark.parametrize("policy,gran", [(1, 0), (2, 1), (0, 1), (3, 0)])
def test_push_eviction_policies(policy, gran):
    """The fused (peer-memory) eviction selection under every policy and both granularities
    equals one unsharded cache's eviction, over several rounds."""
    from paper_2312_04429_b200 import binding as B, sharded as S
    n = 900
    emb, cl = synth.entries(n, seed=60 + policy)
    single = B.NirvanaCache(entry_capacity=n, dim=768, latent_bytes=0, evict_granularity=gran)
    vs = S.VirtualShards(3, entry_capacity=n, dim=768, latent_bytes=0, push_max_nb=64, push_max_topk=1,
                         evict_granularity=gran)
    for c in [single] + vs.caches:
        c.set_evict_policy(policy)
    single.insert(torch.from_numpy(emb).cuda())
    vs.insert(torch.from_numpy(emb).cuda())
    for r in range(3):
        q, _, _ = synth.queries(emb, cl, 3 * 48, seed=90 + r)
        qt = torch.from_numpy(q).cuda()
        single.query(qt, latents=False)
        vs.query(qt, latents=False)
        nev = 50 + 40 * r
        e1, d1 = single.evict(nev)
        e2, d2 = vs.evict(nev)
        assert np.array_equal(e1, e2) and np.array_equal(d1, d2), (policy, gran, r)   # global eviction order
