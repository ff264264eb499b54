"""The eviction path's GPU radix sort (cache_debug_sort_u64) against numpy's sort: one key,
one tile, tile boundaries, a ragged multi-tile tail, heavy duplicates, full 64-bit range."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [1, 2, 2047, 2048, 2049, 100_003, 1_000_000])
@pytest.mark.parametrize("kind", ["random", "dups", "evict_like"])
def test_sort_matches_numpy(n, kind):
    from paper_2312_04429_b200 import binding as B
    rng = np.random.default_rng(n)
    if kind == "random":
        k = rng.integers(0, 2**63, n, dtype=np.int64).view(np.uint64) * np.uint64(2) + rng.integers(0, 2, n).astype(np.uint64)
    elif kind == "dups":
        k = rng.integers(0, 7, n).astype(np.uint64) << np.uint64(60)
    else:   # eviction keys: small scores, unique (id, j) below
        sc = rng.integers(0, 3, n).astype(np.uint64)
        idj = rng.permutation(n).astype(np.uint64)
        k = (sc << np.uint64(35)) | idj
    t = torch.from_numpy(k.view(np.int64).copy()).cuda()
    B.debug_sort_u64(t)
    assert np.array_equal(t.cpu().numpy().view(np.uint64), np.sort(k))
