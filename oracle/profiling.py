"""Cache-selector profiling (Alg. 2) -- plain oracle.

TEST INFRASTRUCTURE ONLY: imported by tests/ and nothing in the product path.

Alg. 2, "Cache Selector-Profiling(K, I_K^c, alpha)":
    for K in the K table:
        [I_K] <- model(P_Q, I_K^c, K) for every profiling prompt P_Q   (the images; here their
                                                                      quality is an input)
        min_sim <- min{ sim s | for all I in [I_K]: quality(I) > alpha }  (garbled set notation)
        sim_K_map[K] <- min_sim
The paper's text: "finds the minimum similarity score such that all generated images
are above a quality threshold alpha", used at run time with the strict '>' of Fig. 11.
Reading R25: the threshold of K is the largest similarity among the profiled
pairs whose image failed (quality <= alpha) -- every pair strictly above it passed; if none
failed, the smallest profiled similarity.  Thresholds are then made non-decreasing in K.
The similarity of a profiling prompt is its cosine to its nearest cached prompt (the exact
top-1 of the oracle's scan), clamped to [-1, 1] as the lookup reports it.
"""
import numpy as np


def profile_thresholds(cache, queries, quality, alpha):
    """cache: oracle.OracleCache holding the cached prompts; queries: [b][dim] profiling prompts;
    quality: [num_k][b] quality of prompt i's image at K_j.  Returns (thresholds[num_k], failed[num_k])."""
    res = cache.query(queries, topk=1, want_latents=False, apply_counters=False)
    b = queries.shape[0]
    sims = []                                  # (similarity, i) of prompts with a valid match
    for i in range(b):
        if int(res["status"][i]) != 0 or int(res["ids"][i, 0]) == int(np.uint64(0xFFFFFFFFFFFFFFFF)):
            continue
        sims.append((float(res["scores"][i, 0]), i))
    if not sims:
        raise ValueError("no profiling prompt has a cached neighbour")
    num_k = quality.shape[0]
    thresholds, failed = [], []
    for j in range(num_k):                     # for K in the K table
        worst_fail = None
        for s, i in sims:                      # all images generated at this K
            if not (float(quality[j][i]) > alpha):
                if worst_fail is None or s > worst_fail:
                    worst_fail = s
        if worst_fail is None:
            thresholds.append(min(s for s, _ in sims))
            failed.append(False)
        else:
            thresholds.append(worst_fail)
            failed.append(True)
    for j in range(1, num_k):                  # non-decreasing in K
        if thresholds[j] < thresholds[j - 1]:
            thresholds[j] = thresholds[j - 1]
    return np.array(thresholds, dtype=np.float64), np.array(failed, dtype=bool)
