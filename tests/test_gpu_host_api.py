"""cache_query_batch_host: host queries in, host results out; latents either gathered into a
device buffer (the denoiser's input) or copied back to host memory -- both equal the device
API's results."""
import numpy as np
import pytest
import torch

import synth
from tests.parity import check_batch, gpu_to_numpy

pytestmark = pytest.mark.gpu


def test_host_call_with_device_latent_buffer():
    from paper_2312_04429_b200 import binding as B
    n, L = 900, 1024
    emb, cl = synth.entries(n, seed=51)
    lat = synth.latents_np(np.arange(n), 5, L, seed=51)
    g = B.NirvanaCache(entry_capacity=n, dim=768, latent_bytes=L)
    g.insert(torch.from_numpy(emb).cuda(), torch.from_numpy(lat).cuda())
    q, _, _ = synth.queries(emb, cl, 77, seed=52)
    d = gpu_to_numpy(g.query(torch.from_numpy(q).cuda(), topk=2))
    qh = torch.from_numpy(q).pin_memory()
    dev_lat = torch.zeros((77, L), dtype=torch.uint8, device="cuda")
    out = dict(ids=np.empty((77, 2), np.uint64), scores=np.empty((77, 2), np.float32), k=np.empty(77, np.int32),
               status=np.empty(77, np.int32), latents=dev_lat)
    g.query_host(qh, topk=2, out=out)
    assert np.array_equal(out["ids"], d["ids"]) and np.array_equal(out["scores"], d["scores"])
    assert np.array_equal(out["k"], d["k"]) and np.array_equal(out["status"], d["status"])
    got = dev_lat.cpu().numpy()
    hit = d["k"] > 0
    assert np.array_equal(got[hit], d["latents"][hit]) and not got[~hit].any()
    h = g.query_host(np.ascontiguousarray(q), topk=2)            # host latent buffer
    assert np.array_equal(h["latents"][hit], d["latents"][hit])


@pytest.mark.parametrize("b", [2048, 3000])
def test_host_call_split_upload_equals_device(oracle_mod, b):
    """b >= 2048: the upload is split into 4 slices (ragged last slice at b=3000) that overlap
    the scan.  Results equal the device call's, and the batch is ONE tick of the LRU clock
    (R13): LRU eviction after the call matches the oracle's, which ticks once per batch."""
    from paper_2312_04429_b200 import binding as B
    n, L = 1500, 256
    emb, cl = synth.entries(n, seed=b)
    lat = synth.latents_np(np.arange(n), 5, L, seed=b)
    mk = lambda: B.NirvanaCache(entry_capacity=n, latent_capacity=5 * n, dim=768, latent_bytes=L)
    g, gd = mk(), mk()
    for c in (g, gd):
        c.set_evict_policy(B.POLICY_LRU)
        c.insert(torch.from_numpy(emb).cuda(), torch.from_numpy(lat).cuda())
    o = oracle_mod.OracleCache(dim=768, entry_capacity=n, latent_capacity=5 * n, latent_bytes=L)
    o.insert(emb, latents=lat)
    q, _, _ = synth.queries(emb, cl, b, seed=b + 1)
    d = gpu_to_numpy(gd.query(torch.from_numpy(q).cuda(), topk=4))
    dev_lat = torch.zeros((b, L), dtype=torch.uint8, device="cuda")
    out = dict(ids=np.empty((b, 4), np.uint64), scores=np.empty((b, 4), np.float32), k=np.empty(b, np.int32),
               status=np.empty(b, np.int32), latents=dev_lat)
    g.query_host(torch.from_numpy(q).pin_memory(), topk=4, out=out)
    for key in ("ids", "scores", "k", "status"):
        assert np.array_equal(out[key], d[key]), key
    hit = d["k"] > 0
    assert np.array_equal(dev_lat.cpu().numpy()[hit], d["latents"][hit])
    check_batch(d, o, q, 4, expected_latent=None)            # oracle: same access, one clock tick
    q2, _, _ = synth.queries(emb, cl, 64, seed=b + 2)        # a second (unsplit) batch on all three
    check_batch(gpu_to_numpy(g.query(torch.from_numpy(q2).cuda(), topk=1, latents=False)), o, q2, 1,
                expected_latent=None)
    gd.query(torch.from_numpy(q2).cuda(), topk=1, latents=False)
    ev, dirty = g.evict(900)
    rc, oev, od = o.evict(900, policy=oracle_mod.LRU)
    assert rc == 0 and np.array_equal(ev, oev) and np.array_equal(dirty, od)
    evd, _ = gd.evict(900)
    assert np.array_equal(ev, evd)


def test_pipelined_submit_complete_matches_device_call(oracle_mod):
    """cache_query_submit / _complete (two slots, uploads on the copy stream): every batch's
    ids / scores / K / status and gathered states equal the device call's for the same cache
    state; one LRU clock tick per batch (the oracle ticks once per batch too)."""
    import torch
    from paper_2312_04429_b200 import binding as B
    n, b, L = 3000, 700, 256
    emb, cl = synth.entries(n, seed=81)
    lat = synth.latents_np(np.arange(n), 5, L, seed=81)
    caches = []
    for _ in range(2):
        g = B.NirvanaCache(entry_capacity=n, dim=768, latent_bytes=L)
        g.set_evict_policy(1)
        g.insert(torch.from_numpy(emb).cuda(), torch.from_numpy(lat).cuda())
        caches.append(g)
    pipe, ref = caches
    qs = [synth.queries(emb, cl, b, seed=90 + i)[0] for i in range(5)]
    qh = [torch.from_numpy(q).pin_memory() for q in qs]
    lats = [torch.empty((b, L), dtype=torch.uint8, device="cuda") for _ in range(2)]
    outs = [dict(ids=torch.empty((b, 1), dtype=torch.int64), scores=torch.empty((b, 1), dtype=torch.float32),
                 k=torch.empty(b, dtype=torch.int32), status=torch.empty(b, dtype=torch.int32)) for _ in range(2)]
    pipe.submit(0, qh[0], 1, lats[0])
    for i in range(5):
        if i + 1 < 5:
            pipe.submit((i + 1) % 2, qh[i + 1], 1, lats[(i + 1) % 2])
        o = pipe.complete(i % 2, outs[i % 2])
        r = ref.query(torch.from_numpy(qs[i]).cuda(), topk=1)
        assert np.array_equal(o["ids"].numpy(), r["ids"].cpu().numpy())
        assert np.array_equal(o["k"].numpy(), r["k"].cpu().numpy())
        assert np.array_equal(o["scores"].numpy().view(np.uint32), r["scores"].cpu().numpy().view(np.uint32))
        hit = r["k"].cpu().numpy() > 0
        assert np.array_equal(lats[i % 2].cpu().numpy()[hit], r["latents"].cpu().numpy()[hit])
    with pytest.raises(B.CacheError):
        pipe.complete(0, outs[0])            # nothing pending
    assert np.array_equal(pipe.evict(2000)[0], ref.evict(2000)[0])   # same LRU clocks
