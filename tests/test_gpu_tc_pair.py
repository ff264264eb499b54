"""The CTA-pair (cta_group::2) scan against the single-CTA scan and the oracle."""
import numpy as np
import pytest
import torch

import synth
from tests.parity import check_batch, gpu_to_numpy

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,b", [(3000, 300), (1000, 129), (777, 256), (5000, 1024)])
def test_pair_equals_single_cta(oracle_mod, n, b):
    from paper_2312_04429_b200 import binding as B
    emb, cl = synth.entries(n, seed=n + b)
    g = B.NirvanaCache(entry_capacity=n, latent_capacity=5 * n, dim=768, latent_bytes=0)
    g.insert(torch.from_numpy(emb).cuda())
    q, _, _ = synth.queries(emb, cl, b, seed=b)
    qt = torch.from_numpy(q).cuda()
    g.set_scorer(B.SCORER_TC_SINGLE)
    d1 = B.debug_tc_scores(g, qt).cpu()
    a = gpu_to_numpy(g.query(qt, topk=4, latents=False))
    g.set_scorer(B.SCORER_AUTO)                                   # b > 128 -> CTA pairs
    d2 = B.debug_tc_scores(g, qt).cpu()
    p = gpu_to_numpy(g.query(qt, topk=4, latents=False))
    assert torch.equal(torch.isnan(d1), torch.isnan(d2))
    m = ~torch.isnan(d1)
    assert (d1[m] - d2[m]).abs().max().item() < 1e-6
    assert np.array_equal(a["k"], p["k"]) and np.array_equal(a["ids"], p["ids"])
    o = oracle_mod.OracleCache(dim=768, entry_capacity=n)
    o.insert(emb)
    check_batch(p, o, q, 4, adopt=False)
