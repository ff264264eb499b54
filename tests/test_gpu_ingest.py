"""Ingest normalisation at volume: stored bf16 rows equal the oracle's plain bf16_RNE(x / ||x||)
with the index-order fp64 norm (R2) bit for bit, up to the proved summation-order accept set
(tests/parity.py check_stored_row: a component may differ only where the exact quotient lies
within the fp64 error bound of a bf16 midpoint; the count is reported and expected 0) --
2,000 of 20,000 rows of mixed magnitudes, fp32 and bf16 inputs, plus rows whose quotients lie
close to bf16 rounding midpoints (the kernel's exact-division fallback path)."""
import numpy as np
import pytest
import torch

import synth
from tests.parity import check_stored_row

pytestmark = pytest.mark.gpu


def _bits(x):
    return (x.astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)


def test_stored_rows_bit_identical_at_volume(oracle_mod):
    from paper_2312_04429_b200 import binding as B
    n = 20_000
    emb, _ = synth.entries(n, seed=123)
    rng = np.random.default_rng(0)
    emb *= np.float32(10.0) ** rng.integers(-6, 6, size=(n, 1)).astype(np.float32)
    # rows with ||x|| = 2^k exactly whose components are bf16 rounding midpoints:
    # x = 2^k * (1 + 2^-8, ...)?  Use (m, m, ..., r) with sum of squares 4^k: 16 copies of
    # a = 1 + 2^-8 scaled so that 16 a^2 + r^2 = 64 -> r chosen exactly representable
    mid = np.float32(1.0 + 2.0 ** -8)            # midpoint between bf16 1.0 and 1.0078125
    for i in range(50):
        row = np.zeros(768, np.float32)
        row[:16] = mid
        rest = 64.0 - 16.0 * float(mid) ** 2      # = 64 - 16(1 + 2^-7 + 2^-16) exactly in fp64
        row[16] = np.float32(np.sqrt(rest))      # inexact: the row norm is then ~8, not exactly
        emb[i] = row
    g = B.NirvanaCache(entry_capacity=n, latent_capacity=5 * n, dim=768, latent_bytes=0)
    g.insert(torch.from_numpy(emb).cuda())
    accepted = 0
    for i in list(range(60)) + list(rng.choice(n, 2000, replace=False)):
        _, y = oracle_mod.normalise(emb[i].astype(np.float64))
        accepted += check_stored_row(g.row_bf16(int(i)), emb[i], y)
    print(f"stored-row accept-set components (fp32 inputs): {accepted}")
    assert accepted == 0
    # bf16 inputs go through the same rule
    eb = torch.from_numpy(emb[:300]).to(torch.bfloat16)
    g2 = B.NirvanaCache(entry_capacity=300, latent_capacity=1500, dim=768, latent_bytes=0)
    g2.insert(eb.cuda())
    ebits = eb.view(torch.int16).numpy().view(np.uint16)
    o = oracle_mod.OracleCache(dim=768, entry_capacity=300)
    o.insert(ebits, emb_is_bf16=True)
    xb = eb.float().numpy()
    assert sum(check_stored_row(g2.row_bf16(i), xb[i], o.row(i)) for i in range(300)) == 0
