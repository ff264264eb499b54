"""The shared seeded input generator: determinism and numpy/torch agreement (no GPU)."""
import numpy as np
import pytest

import synth


def test_entries_deterministic_and_unit():
    a, ca = synth.entries(500, seed=9)
    b, cb = synth.entries(500, seed=9)
    assert np.array_equal(a, b) and np.array_equal(ca, cb)
    n = np.sqrt((a.astype(np.float64) ** 2).sum(1))
    assert np.allclose(n, 1.0, atol=1e-5)


def test_query_similarity_mixture():
    emb, cl = synth.entries(2000, seed=3)
    q, anchor, t = synth.queries(emb, cl, 4000, seed=3)
    cos = (q.astype(np.float64) * emb[anchor]).sum(1)
    assert np.abs(cos - t).mean() < 0.01              # target cosine to the anchor is realised
    assert 0.09 < (t < 0.65).mean() < 0.15            # ~12% below the lowest threshold


def test_latents_numpy_torch_agree():
    torch = pytest.importorskip("torch")
    rows = np.arange(37, 37 + 9)
    a = synth.latents_np(rows, 5, 256, seed=1234)
    b = synth.latents_torch(37, 9, 5, 256, seed=1234, device="cpu").numpy()
    assert np.array_equal(a, b)
    words = a.view(np.uint32).reshape(9, 5, 64)
    assert (words[:, :, 0] == rows[:, None]).all() and (words[:, :, 2] == np.arange(5)).all()
    assert (words[:, :, 3] == synth.MAGIC).all()
