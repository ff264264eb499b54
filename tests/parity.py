"""Parity harness: compare one GPU lookup batch with the fp64 oracle (SURVEY 8(c) contract).

Accept rules, tau = the strict tier 2^-12 unless a test says
otherwise:
  * every rank t < k: if the oracle gaps on both sides of rank t (s_{t-1} - s_t and
    s_t - s_{t+1}) are >= tau, the GPU id at rank t must equal the oracle's; otherwise the GPU
    id must lie in the oracle's tau-band around s_t (|s(gpu id) - s_t| <= tau).  Rank 0 with a
    gap below tau is an "exempt" query.  The GPU lists as many ids as the oracle (pads with
    UINT64_MAX when fewer than k entries are live), all distinct, scores non-increasing.
  * score at every rank: |gpu score - clamp(oracle fp64 score of that GPU id)| <= tau_score
    (1e-4: the fp32-accumulation bound of DESIGN 4)
  * K: equals the Fig. 11 map + hole rule applied to the oracle's fp64 score of the GPU's
    rank-0 entry; if that score is within tau of a threshold either adjacent bucket is accepted
  * latent bytes: bit-exact equal to the stored state (entry, K) whenever K > 0
  * counters: the oracle adopts each accepted GPU (entry, K) so multi-round state stays equal
  * stored rows (check_stored_row): bit-identical to the oracle's bf16_RNE(x / ||x||) except
    where the exact quotient lies within the two summation orders' fp64 error bound of a bf16
    rounding midpoint (proved per component with 60-digit decimal arithmetic, counted)
"""
from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor
from decimal import Decimal, getcontext
import os

import numpy as np

TAU = 2e-3            # north_star contract tier
TAU_STRICT = 2 ** -12  # provable fp32-accumulation margin; the gate the tests assert
TAU_SCORE = 1e-4      # score agreement: gamma_768 ~ 4.6e-5, x2 for the two inv-norm multiplies
NO_ID = 0xFFFFFFFFFFFFFFFF


def hole_resolve(kstar: int, mask: int, k_values) -> int:
    """Largest present K <= K* (P:616-619); 0 if none."""
    best = 0
    for j, k in enumerate(k_values):
        if (mask >> j) & 1 and k <= kstar:
            best = k
    return best


def _oracle_query_rows(orc, q, rows, topk, threads=None):
    """The oracle's read-only query (apply_counters=False) of the sampled rows, split over host
    threads (ctypes releases the GIL, so the unchanged C oracle runs on every core)."""
    rows = list(rows)
    nt = threads or max(1, min(len(os.sched_getaffinity(0)), 32))
    chunks = [rows[i::nt] for i in range(nt) if rows[i::nt]]
    with ThreadPoolExecutor(max_workers=len(chunks) or 1) as ex:
        parts = list(ex.map(lambda c: orc.query(q[c], topk=topk, want_latents=False, apply_counters=False),
                            chunks))
    ids = np.empty((len(rows), topk), np.uint64)
    raw = np.empty((len(rows), topk), np.float64)
    pos = {r: i for i, r in enumerate(rows)}
    for c, p in zip(chunks, parts):
        for j, r in enumerate(c):
            ids[pos[r]] = p["ids"][j]
            raw[pos[r]] = p["raw"][j]
    return dict(ids=ids, raw=raw)


def check_batch(gpu: dict, orc, q: np.ndarray, topk: int, expected_latent=None, tau: float = TAU_STRICT,
                tau_score: float = TAU_SCORE, adopt: bool = True, rows=None):
    """gpu: dict of numpy arrays ids[b][topk] (u64), scores[b][topk], k[b], latents[b][L] or None.
    expected_latent(id, K) -> bytes of the stored state.  rows: subset of query rows to check.
    Returns a report dict; raises AssertionError on a contract violation."""
    b = q.shape[0]
    rows = list(range(b)) if rows is None else [int(r) for r in rows]
    ores = _oracle_query_rows(orc, q, rows, topk + 1)
    rep = dict(checked=0, exempt=0, exempt_contract=0, rank_band=0, k_adjacent=0, max_dscore=0.0, hits=0,
               ranks_checked=0)
    acc_ids, acc_k = [], []
    kv = orc.k_values
    for oi, i in enumerate(rows):
        rep["checked"] += 1
        gid = int(gpu["ids"][i, 0])
        gk = int(gpu["k"][i])
        oids = [int(x) for x in ores["ids"][oi]]
        osc = [float(x) for x in ores["raw"][oi]]
        n_o = sum(1 for x in oids[:topk] if x != NO_ID)
        gids = [int(x) for x in gpu["ids"][i]]
        n_g = sum(1 for x in gids if x != NO_ID)
        assert n_g == n_o and all(x == NO_ID for x in gids[n_g:]), \
            f"row {i}: gpu lists {n_g} ids, oracle {n_o}"
        if n_o == 0:
            assert gk == 0, f"row {i}: oracle has no entry, gpu K {gk}"
            continue
        assert len(set(gids[:n_g])) == n_g, f"row {i}: duplicate ids {gids}"
        sc = gpu["scores"][i, :n_g]
        assert all(sc[t] >= sc[t + 1] for t in range(n_g - 1)), f"row {i}: scores not best-first {sc}"
        s_gpu_entry = []
        for t in range(n_g):
            rep["ranks_checked"] += 1
            up = osc[t - 1] - osc[t] if t > 0 else np.inf
            down = osc[t] - osc[t + 1] if (t + 1 < len(oids) and oids[t + 1] != NO_ID) else np.inf
            g_t = gids[t]
            sg = osc[t] if g_t == oids[t] else orc.score_id(q[i], g_t)
            if up >= tau and down >= tau:
                assert g_t == oids[t], f"row {i} rank {t}: gpu id {g_t} != oracle {oids[t]} " \
                                       f"(gaps {up:.3g} / {down:.3g})"
            elif g_t != oids[t]:
                rep["rank_band"] += 1
                assert abs(sg - osc[t]) <= tau, f"row {i} rank {t}: gpu id {g_t} (s={sg}) outside the " \
                                                f"tau band of the oracle's s_t={osc[t]}"
            c = min(max(sg, -1.0), 1.0)
            d = abs(float(gpu["scores"][i, t]) - c)
            rep["max_dscore"] = max(rep["max_dscore"], d)
            assert d <= tau_score, f"row {i} rank {t}: score {gpu['scores'][i, t]} vs oracle {c}"
            s_gpu_entry.append(sg)
        gap1 = osc[0] - osc[1] if oids[1] != NO_ID else np.inf
        if gap1 < tau:
            rep["exempt"] += 1
        if gap1 < TAU:
            rep["exempt_contract"] += 1
        sg = s_gpu_entry[0]
        _, mask = orc.meta(gid)
        want = hole_resolve(orc.select_k(sg), mask, kv)
        if gk != want:
            alt = {hole_resolve(orc.select_k(sg + d), mask, kv) for d in (-tau, tau)}
            assert gk in alt, f"row {i}: K {gk} != {want} (score {sg})"
            rep["k_adjacent"] += 1
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


# ----------------------------------------------------------------------------------------
# stored rows: bit-identical up to a proved accept set
# ----------------------------------------------------------------------------------------
def _bf16_value(bits: int) -> float:
    return float(np.array([int(bits) << 16], np.uint32).view(np.float32)[0])


def check_stored_row(gpu_bits: np.ndarray, x: np.ndarray, oracle_y: np.ndarray) -> int:
    """gpu_bits: the GPU's stored bf16 bit patterns of one row; x: the input row (fp32 or the
    fp64 values of bf16 inputs); oracle_y: the oracle's stored fp64 values (its plain
    index-order normalisation).

    The kernel sums the squares in another order, so its norm may differ from the oracle's in
    the last bits.  Both quotients are within delta = ((dim-1)/2 + 2) u (u = 2^-53: the sum of
    dim positive exact squares in any order, then sqrt, then the division) of the exact
    x_i / ||x||, so the two RNE roundings can differ only where a bf16 rounding midpoint lies
    within delta of the exact quotient.  Every differing component must be such a case: the
    two values must be the adjacent bf16 neighbours of the exact quotient and their midpoint
    within 2 delta |q_i| of it (60-digit decimal).  Returns the number of such components."""
    y_bits = (np.asarray(oracle_y, np.float64).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
    gpu_bits = np.asarray(gpu_bits, np.uint16)
    diff = np.nonzero(gpu_bits != y_bits)[0]
    if len(diff) == 0:
        return 0
    getcontext().prec = 60
    dim = len(x)
    xs = [Decimal(float(v)) for v in x]
    nrm = sum(v * v for v in xs).sqrt()
    delta = Decimal(2 * ((dim - 1) / 2 + 2)) * Decimal(2) ** -53
    for i in diff:
        qi = xs[i] / nrm
        a, c = _bf16_value(gpu_bits[i]), _bf16_value(y_bits[i])
        lo, hi = min(a, c), max(a, c)
        # adjacent bf16 values: one bf16 quantum apart (same sign), bracketing the exact value
        step = np.uint16(abs(int(gpu_bits[i]) - int(y_bits[i])))
        assert step == 1 and (gpu_bits[i] & 0x8000) == (y_bits[i] & 0x8000), \
            f"component {i}: gpu {a} vs oracle {c} are not adjacent bf16 values"
        assert Decimal(lo) <= qi <= Decimal(hi), f"component {i}: {a}, {c} do not bracket {qi}"
        mid = (Decimal(lo) + Decimal(hi)) / 2
        assert abs(qi - mid) <= delta * abs(qi), \
            f"component {i}: exact {qi} is {abs(qi - mid) / abs(qi):.3e} (rel) from the midpoint, " \
            f"beyond the summation-order bound {delta:.3e}: the GPU rounding is wrong"
    return len(diff)


def gpu_to_numpy(out: dict) -> dict:
    r = dict(ids=out["ids"].cpu().numpy().view(np.uint64), scores=out["scores"].cpu().numpy(),
             k=out["k"].cpu().numpy(), status=out["status"].cpu().numpy())
    r["latents"] = out["latents"].cpu().numpy() if out.get("latents") is not None else None
    return r
