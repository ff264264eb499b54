"""Failure detection on the multi-rank path: a rank that does not publish within the
peer timeout makes the push exchange fail CLEANLY -- the waiting rank gets CACHE_E_NCCL (from
cache_push_status and every later cache_push_* call), no kernel touches peer memory after the
failure, the CUDA context stays usable (local caches keep answering), and nothing hangs or
traps.  (A peer is stalled, not killed: a killed exporter's IPC memory would be freed under the
survivor's mappings, which no library can make safe.)"""
import os
import socket
import time

import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


def _local_cache_still_works(B):
    emb, cl = synth.entries(300, seed=3)
    plain = B.NirvanaCache(entry_capacity=300, dim=768, latent_bytes=0)
    plain.insert(torch.from_numpy(emb).cuda())
    out = plain.query(torch.from_numpy(emb[:16]).cuda(), latents=False)
    torch.cuda.synchronize()
    assert np.array_equal(out["ids"][:, 0].cpu().numpy(), np.arange(16))


def test_stalled_virtual_rank_reports_nccl_status():
    from paper_2312_04429_b200 import binding as B, sharded as S
    n, nb = 400, 32
    emb, cl = synth.entries(n, seed=8)
    vs = S.VirtualShards(2, entry_capacity=n, dim=768, latent_bytes=0, push_max_nb=nb, push_max_topk=1)
    vs.insert(torch.from_numpy(emb).cuda())
    c0 = vs.caches[0]
    c0.set_peer_timeout(300)
    q = torch.from_numpy(synth.queries(emb, cl, nb, seed=9)[0]).cuda()
    t0 = time.perf_counter()
    c0.push_queries(q)             # rank 1 never publishes its queries
    c0.push_scan(nb, 1)
    out = c0.alloc_outputs(nb, 1, latents=False)
    try:
        c0.push_merge(nb, 1, out)
    except B.CacheError as e:      # the host may already have seen the timeout
        assert e.code == B.E_NCCL
    with pytest.raises(B.CacheError) as ei:
        c0.push_status()
    assert ei.value.code == B.E_NCCL and "peer" in str(ei.value)
    assert time.perf_counter() - t0 < 30
    with pytest.raises(B.CacheError) as ei:   # the handle stays failed
        c0.push_queries(q)
    assert ei.value.code == B.E_NCCL
    _local_cache_still_works(B)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _proc(rank, port, ret):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        torch.cuda.set_device(0)
        from paper_2312_04429_b200 import binding as B, sharded as S
        n, nb = 400, 16
        emb, cl = synth.entries(n, seed=12)
        comm = S.TorchComm(device="cpu")
        sc = S.ShardedCache(comm, entry_capacity=n, dim=768, latent_bytes=0, push_max_nb=nb, push_max_topk=1)
        sc.insert(torch.from_numpy(emb).cuda())
        sc.cache.set_peer_timeout(500)
        q = torch.from_numpy(synth.queries(emb, cl, 2 * nb, seed=13)[0][rank * nb:(rank + 1) * nb]).cuda()
        out = sc.alloc_outputs(nb, 1, latents=False)
        sc.query_into(q, out)        # one good batch on both ranks
        sc.cache.push_status()
        if rank == 1:                # rank 1 stalls: it stops serving until rank 0 is done
            dist.barrier()
            ret[rank] = True
            return
        code = None
        try:
            sc.query_into(q, out)
            sc.cache.push_status()
        except B.CacheError as e:
            code = e.code
        ok = code == B.E_NCCL
        _local_cache_still_works(B)
        ret[rank] = ok
        dist.barrier()
    except Exception as e:           # noqa: BLE001
        ret[rank] = repr(e)
    finally:
        dist.destroy_process_group()


def test_stalled_process_reports_nccl_status():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    port = _free_port()
    mgr = ctx.Manager()
    ret = mgr.dict()
    procs = [ctx.Process(target=_proc, args=(r, port, ret)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    for p in procs:
        if p.is_alive():
            p.kill()
    assert dict(ret) == {0: True, 1: True}, dict(ret)
