"""Parity harness: compare one GPU lookup batch with the fp64 oracle (SURVEY 8(c) contract).

Accept rules:
  * entry: if the oracle's top-1/top-2 gap >= tau the GPU entry must equal the oracle top-1;
    otherwise it must be in {e : s_e >= s_1 - tau}  (an "exempt" query)
  * K: equals the Fig. 11 map + hole rule applied to the oracle's fp64 score of the GPU's entry;
    if that score is within tau of a threshold either adjacent bucket is accepted
  * score: |gpu score - clamp(oracle score of the GPU entry)| <= tau_score
  * latent bytes: bit-exact equal to the stored state (entry, K) whenever K > 0
  * counters: the oracle adopts each accepted GPU (entry, K) so multi-round state stays equal
"""
from __future__ import annotations

import numpy as np

TAU = 2e-3            # north_star contract tier
TAU_STRICT = 2 ** -12  # provable fp32-accumulation margin


def hole_resolve(kstar: int, mask: int, k_values) -> int:
    """Largest present K <= K* (P:616-619); 0 if none."""
    best = 0
    for j, k in enumerate(k_values):
        if (mask >> j) & 1 and k <= kstar:
            best = k
    return best


def check_batch(gpu: dict, orc, q: np.ndarray, topk: int, expected_latent=None, tau: float = TAU,
                tau_score: float = TAU, adopt: bool = True, rows=None):
    """gpu: dict of numpy arrays ids[b][topk] (u64), scores[b][topk], k[b], latents[b][L] or None.
    expected_latent(id, K) -> bytes of the stored state.  rows: subset of query rows to check.
    Returns a report dict; raises AssertionError on a contract violation."""
    b = q.shape[0]
    rows = range(b) if rows is None else rows
    ores = orc.query(q[list(rows)], topk=max(topk, 2), want_latents=False, apply_counters=False)
    rep = dict(checked=0, exempt=0, exempt_strict=0, k_adjacent=0, max_dscore=0.0, hits=0)
    acc_ids, acc_k = [], []
    for oi, i in enumerate(rows):
        rep["checked"] += 1
        gid = int(gpu["ids"][i, 0])
        gk = int(gpu["k"][i])
        s1 = ores["raw"][oi, 0]
        if int(ores["ids"][oi, 0]) == int(np.uint64(0xFFFFFFFFFFFFFFFF)):
            assert gid == 0xFFFFFFFFFFFFFFFF and gk == 0, f"row {i}: oracle has no entry, gpu {gid}"
            continue
        s2 = ores["raw"][oi, 1] if np.isfinite(ores["raw"][oi, 1]) else -np.inf
        oid = int(ores["ids"][oi, 0])
        if s1 - s2 >= tau:
            assert gid == oid, f"row {i}: gpu entry {gid} != oracle {oid} (gap {s1 - s2:.3g})"
        else:
            rep["exempt"] += 1
            if gid != oid:
                sg = orc.score_id(q[i], gid)
                assert sg >= s1 - tau, f"row {i}: gpu entry {gid} score {sg} not within tau of {s1}"
        if s1 - s2 < TAU_STRICT:
            rep["exempt_strict"] += 1
        sg = s1 if gid == oid else orc.score_id(q[i], gid)
        c = min(max(sg, -1.0), 1.0)
        rep["max_dscore"] = max(rep["max_dscore"], abs(float(gpu["scores"][i, 0]) - c))
        assert abs(float(gpu["scores"][i, 0]) - c) <= tau_score, f"row {i}: score {gpu['scores'][i, 0]} vs {c}"
        _, mask = orc.meta(gid)
        kv = orc.k_values
        want = hole_resolve(orc.select_k(sg), mask, kv)
        if gk != want:
            alt = {hole_resolve(orc.select_k(sg + d), mask, kv) for d in (-tau, tau)}
            assert gk in alt, f"row {i}: K {gk} != {want} (score {sg})"
            rep["k_adjacent"] += 1
        # top-k list: ids must be distinct and scores non-increasing
        ids_row = [int(x) for x in gpu["ids"][i] if int(x) != 0xFFFFFFFFFFFFFFFF]
        assert len(set(ids_row)) == len(ids_row)
        sc = gpu["scores"][i, : len(ids_row)]
        assert all(sc[t] >= sc[t + 1] for t in range(len(sc) - 1))
        if gk > 0:
            rep["hits"] += 1
            if expected_latent is not None and gpu.get("latents") is not None:
                exp = expected_latent(gid, gk)
                assert np.array_equal(gpu["latents"][i], exp), f"row {i}: latent bytes differ"
        acc_ids.append(gid)
        acc_k.append(gk)
    if adopt:   # one GPU query batch = one record_access call = one tick of the LRU clock
        assert orc.record_access(np.array(acc_ids, np.uint64), np.array(acc_k, np.int32)) == 0
    return rep


def gpu_to_numpy(out: dict) -> dict:
    r = dict(ids=out["ids"].cpu().numpy().view(np.uint64), scores=out["scores"].cpu().numpy(),
             k=out["k"].cpu().numpy(), status=out["status"].cpu().numpy())
    r["latents"] = out["latents"].cpu().numpy() if out.get("latents") is not None else None
    return r
