"""The tcgen05 main loop on its own: dense scan values vs a plain PyTorch fp32 reference."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def B():
    from paper_2312_04429_b200 import binding
    return binding


def _stored(cache, n):
    rows = np.stack([cache.row_bf16(i) for i in range(n)])
    return torch.from_numpy((rows.astype(np.uint32) << 16).view(np.float32))


@pytest.mark.parametrize("n,b,dim", [(256, 128, 768), (1000, 64, 768), (777, 130, 768), (300, 3, 64),
                                     (2048, 300, 1024), (513, 257, 128)])
def test_tc_dense_matches_torch_fp32(B, oracle_mod, n, b, dim):
    emb, cl = synth.entries(n, seed=n, dim=dim)
    g = B.NirvanaCache(entry_capacity=n, dim=dim, latent_bytes=0, latent_capacity=5 * n)
    g.insert(torch.from_numpy(emb).cuda())
    q, _, _ = synth.queries(emb, cl, b, seed=b, )
    dense = B.debug_tc_scores(g, torch.from_numpy(q).cuda()).cpu()
    x = _stored(g, n).double()
    qn = torch.from_numpy(np.stack([oracle_mod.normalise(r.astype(np.float64))[1] for r in q]))
    inv = 1.0 / torch.sqrt((x * x).sum(1))
    ref = (qn.float() @ x.float().T).double() * inv          # plain torch fp32 GEMM, fp64 scale
    got = dense[:, :n].double()
    assert torch.isfinite(got).all()
    err = (got - ref).abs().max().item()
    assert err < 2e-5, err
    assert torch.isnan(dense[:, n:]).all()                      # empty slots carry NaN


def test_tc_single_tile_exact_on_dyadic_data(B):
    """Entries/queries with few-bit dyadic components: every product and partial sum is exact
    in fp32, so the tensor-core result must equal the exact integer dot product."""
    rng = np.random.default_rng(0)
    n, b, dim = 256, 128, 768
    e = rng.integers(-3, 4, size=(n, dim)).astype(np.float32)
    q = rng.integers(-3, 4, size=(b, dim)).astype(np.float32)
    e[:, 0] = 64.0   # dominant component so the normalised row is a power-of-two scale of e
    g = B.NirvanaCache(entry_capacity=n, dim=dim, latent_bytes=0, latent_capacity=5 * n)
    g.insert(torch.from_numpy(e).cuda())
    dense = B.debug_tc_scores(g, torch.from_numpy(q).cuda()).cpu().double()
    x = _stored(g, n).double()
    qs = torch.from_numpy(np.stack([(np.asarray(q[i], np.float64)) for i in range(b)]))
    # reference on the stored (bf16) values, exact in fp64
    from oracle import normalise
    qn = torch.from_numpy(np.stack([normalise(r.astype(np.float64))[1] for r in q]))
    inv = (1.0 / torch.sqrt((x * x).sum(1))).float().double()
    ref = (qn @ x.T)
    assert torch.allclose(dense, (ref.float().double() * inv).float().double(), atol=1e-6, rtol=1e-6)
