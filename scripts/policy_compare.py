"""Directional reproduction of the paper's policy comparison (Table 3; SPEC
acceptance #6) on a synthetic skewed-similarity stream, through the CUDA library.

python scripts/policy_compare.py [--universe 200000] [--batches 300] [--batch 512]
Prints one JSON line per (capacity, policy): hit-rate, compute savings f_C, latency model.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_2312_04429_b200 import binding as B  # noqa: E402
from paper_2312_04429_b200.serving import GpuCache, LatencyParams, ServingLoop  # noqa: E402

NAMES = {0: "LCBFU", 1: "LRU", 2: "LFU", 3: "FIFO"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--universe", type=int, default=200_000)
    ap.add_argument("--batches", type=int, default=300)
    ap.add_argument("--batch", type=int, default=512)
    ap.add_argument("--capacities", default="2000,8000,32000")
    a = ap.parse_args()
    universe, cl = synth.entries(a.universe, seed=2024)
    streams = [synth.queries(universe, cl, a.batch, seed=9000 + i)[0] for i in range(a.batches)]
    for cap in [int(x) for x in a.capacities.split(",")]:
        for policy in (0, 1, 2, 3):
            g = B.NirvanaCache(entry_capacity=cap, latent_capacity=5 * cap, dim=768, latent_bytes=0)
            g.set_evict_policy(policy)
            loop = ServingLoop(GpuCache(g), synth.K_VALUES, LatencyParams())
            for q in streams:
                loop.step(q)
            s = loop.report.summary(loop.lat)
            print(json.dumps(dict(capacity_entries=cap, capacity_states=5 * cap, policy=NAMES[policy],
                                  hit_rate=s["hit_rate"], f_c=s["f_c"], h_opt=s["h_opt"],
                                  mean_latency_s=s["mean_latency_s"],
                                  latency_reduction=s["latency_reduction_vs_scratch"],
                                  evicted=s["evicted_items"], requests=s["requests"])), flush=True)


if __name__ == "__main__":
    main()
