"""Timings of the widened rows on the C2 cache (100K entries x 768): match-predictor training
(NEXT-3, cache_predictor_train) and per-query prediction (cache_predict), and cache-selector
profiling (NEXT-4, cache_profile_thresholds).  CUDA events on the launching stream, median
of several runs; synthetic inputs from synth/.  Diagnostic, prints one JSON line."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2312_04429_b200 import binding as B  # noqa: E402


def ev_ms(fn, reps):
    out = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        fn()
        e.record()
        e.synchronize()
        out.append(s.elapsed_time(e))
    return statistics.median(out)


def main():
    n, b = 100_000, 4096
    emb, cl = synth.entries(n, seed=1000)
    g = B.NirvanaCache(entry_capacity=n, dim=768, latent_bytes=0, latent_capacity=5 * n)
    g.insert(torch.from_numpy(emb).cuda())
    q = torch.from_numpy(synth.queries(emb, cl, b, seed=1001)[0]).cuda()
    g.train_predictor(epochs=50)   # warm-up
    train = ev_ms(lambda: g.train_predictor(epochs=50), 3)
    g.predict(q)
    pred = ev_ms(lambda: g.predict(q), 20)
    quality = torch.rand((5, b), device="cuda", generator=torch.Generator(device="cuda").manual_seed(7))
    g.profile_thresholds(q, quality)
    prof = ev_ms(lambda: g.profile_thresholds(q, quality), 10)
    print(json.dumps(dict(entries=n, predictor_train_ms_50_epochs=train, predictor_train_ms_per_epoch=train / 50,
                          predict_ms_4096=pred, predict_queries_per_s=b / (pred / 1e3),
                          profile_thresholds_ms_4096_prompts=prof,
                          note="CUDA events around each host call (train and profile synchronise internally)")))


if __name__ == "__main__":
    main()
