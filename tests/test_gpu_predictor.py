"""NEXT-3 on the GPU: the predictor trained by the CUDA kernels agrees with the fp64 oracle
trained on the same stored embeddings (model and decisions), and gates queries."""
import numpy as np
import pytest
import torch

import synth
from oracle import predictor as OP
from tests.test_predictor_oracle import _cone

pytestmark = pytest.mark.gpu


def test_gpu_predictor_matches_oracle(oracle_mod):
    from paper_2312_04429_b200 import binding as B
    n = 6000
    X, c = _cone(n, seed=3)
    X = X.astype(np.float32)
    g = B.NirvanaCache(entry_capacity=n, latent_capacity=5 * n, dim=768, latent_bytes=0)
    g.insert(torch.from_numpy(X).cuda())
    o = oracle_mod.OracleCache(dim=768, entry_capacity=n)
    o.insert(X)
    S = np.stack([o.row(i) for i in range(n)])
    S /= np.linalg.norm(S, axis=1, keepdims=True)                  # unit-scaled stored values
    nu, epochs, lr0 = 0.001, 40, 0.5
    w_o, rho_o = OP.train(S, nu=nu, epochs=epochs, lr0=lr0)
    g.train_predictor(nu=nu, epochs=epochs, lr0=lr0)
    w_g, rho_g = g.predictor()
    cos = float(w_g @ w_o / (np.linalg.norm(w_g) * np.linalg.norm(w_o)))
    assert cos > 0.9999 and abs(rho_g - rho_o) < 2e-3 * max(1.0, abs(rho_o)), (cos, rho_g, rho_o)
    rng = np.random.default_rng(4)
    probes = np.vstack([X[:500], -X[:200], rng.standard_normal((300, 768)).astype(np.float32),
                        (X[500:800] + 0.3 * rng.standard_normal((300, 768)).astype(np.float32))])
    flags, margin = g.predict(torch.from_numpy(probes).cuda())
    flags = flags.cpu().numpy().astype(bool)
    Pn = np.stack([oracle_mod.normalise(p.astype(np.float64))[1] for p in probes])
    Pn /= np.linalg.norm(Pn, axis=1, keepdims=True)
    f_o = OP.decision(w_o, rho_o, Pn)
    clear = np.abs(f_o) > 5e-3
    assert np.array_equal(flags[clear], (f_o >= 0)[clear])
    assert flags[:500].mean() >= 0.99 and not flags[500:700].any()
