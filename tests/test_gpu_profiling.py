"""Cache-selector profiling on the GPU (cache_profile_thresholds, Alg. 2) against the oracle:
the exact hand case, random parity, no access counted, and the installed table driving K."""
import numpy as np
import pytest
import torch

import synth
from oracle import profiling
from tests.parity import check_batch, gpu_to_numpy

pytestmark = pytest.mark.gpu


def test_hand_profile_exact_on_gpu():
    from paper_2312_04429_b200 import binding as B
    H = synth.hand_vectors(768)
    g = B.NirvanaCache(entry_capacity=4, dim=768, latent_bytes=0, latent_capacity=20)
    g.insert(torch.from_numpy(H[[1]]).cuda())
    q = torch.from_numpy(H[[0, 2, 4]]).cuda()
    quality = torch.tensor([[0.95, 0.97, 0.99], [0.50, 0.95, 0.99], [0.50, 0.80, 0.99], [0.10, 0.20, 0.90],
                            [0.10, 0.20, 0.30]], dtype=torch.float32, device="cuda")
    thr, failed = g.profile_thresholds(q, quality, alpha=0.9)
    assert list(thr) == [0.75, 0.75, 0.875, 0.921875, 0.921875]
    assert list(failed) == [False, True, True, True, True]
    f, _ = g.meta(0)
    assert not f.any()                                   # profiling counts no access


@pytest.mark.parametrize("n,b", [(2000, 700), (8000, 1200)])
def test_profile_parity_and_install(oracle_mod, n, b):
    from paper_2312_04429_b200 import binding as B
    emb, cl = synth.entries(n, seed=n)
    g = B.NirvanaCache(entry_capacity=n, dim=768, latent_bytes=0, latent_capacity=5 * n)
    g.insert(torch.from_numpy(emb).cuda())
    o = oracle_mod.OracleCache(dim=768, entry_capacity=n)
    o.insert(emb)
    q, _, _ = synth.queries(emb, cl, b, seed=b)
    sims = o.query(q, topk=1, want_latents=False, apply_counters=False)["scores"][:, 0]
    tau = np.array([0.66, 0.77, 0.84, 0.91, 0.96])
    rng = np.random.default_rng(1)
    quality = (0.9 + (sims[None, :] - tau[:, None]) + rng.normal(0, 0.01, (5, b))).astype(np.float32)
    thr, failed = g.profile_thresholds(torch.from_numpy(q).cuda(), torch.from_numpy(quality).cuda(), alpha=0.9)
    othr, ofailed = profiling.profile_thresholds(o, q, quality, 0.9)
    assert np.array_equal(failed, ofailed)
    assert np.abs(thr - othr).max() < 1e-4
    # install the profiled table; lookups then map scores with it (oracle given the same table)
    g.set_thresholds(thr)
    o2 = oracle_mod.OracleCache(dim=768, entry_capacity=n, thresholds=tuple(float(x) for x in thr))
    o2.insert(emb)
    q2, _, _ = synth.queries(emb, cl, 512, seed=b + 1)
    out = gpu_to_numpy(g.query(torch.from_numpy(q2).cuda(), topk=1, latents=False))
    check_batch(out, o2, q2, 1, expected_latent=None)
    with pytest.raises(B.CacheError):
        g.set_thresholds(thr[::-1] if thr[0] < thr[-1] else [0.9, 0.8, 0.7, 0.6, 0.5])
