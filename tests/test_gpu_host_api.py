"""cache_query_batch_host: host queries in, host results out; latents either gathered into a
device buffer (the denoiser's input) or copied back to host memory -- both equal the device
API's results."""
import numpy as np
import pytest
import torch

import synth
from tests.parity import gpu_to_numpy

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
