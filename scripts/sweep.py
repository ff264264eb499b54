"""Batch-size sweep of both scorers on one cache (CUDA-event timing, L2 flushed per step).

python scripts/sweep.py --n 100000 --latents 1 --batches 1,2,4,8,16,32,64,128,256,1024,4096
Prints one JSON object per (scorer, batch) with per-kernel times and roofline fractions.
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2312_04429_b200 import binding as B  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=100_000)
    ap.add_argument("--latents", type=int, default=1)
    ap.add_argument("--batches", default="1,2,4,8,16,32,64,128,256,512,1024,4096")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--scorers", default="stream,tc")
    ap.add_argument("--topks", default="1", help="comma list of topk values (fused top-k width)")
    ap.add_argument("--flush", default="write", choices=["write", "write+read", "none"],
                    help="L2 treatment between steps: write 512 MiB (bench.py's rule; the dirty lines are "
                         "written back during the next step), write then read a second 512 MiB buffer "
                         "(cold and clean), or nothing")
    a = ap.parse_args()
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    n, L = a.n, 32768 if a.latents else 0
    emb, cl = synth.entries(n, seed=1000)
    pres = synth.present_masks(n, seed=1000)
    g = B.NirvanaCache(entry_capacity=n, dim=768, latent_bytes=L, latent_capacity=5 * n)
    for s in range(0, n, 8192):
        m = min(8192, n - s)
        lat = synth.latents_torch(s, m, 5, L, seed=1000, device="cuda") if L else None
        g.insert(torch.from_numpy(emb[s:s + m]).cuda(), lat, present=pres[s:s + m])
        del lat
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    flush2 = torch.ones(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda") if a.flush == "write+read" else None
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    g.set_profile_events(ev)
    bmax = max(int(x) for x in a.batches.split(","))
    qall, _, _ = synth.queries(emb, cl, bmax, seed=1001)
    for scorer in a.scorers.split(","):
        g.set_scorer(B.SCORER_STREAM if scorer == "stream" else B.SCORER_TC)
        for b, topk in [(int(x), int(k)) for x in a.batches.split(",") for k in a.topks.split(",")]:
            if scorer == "stream" and b > 64:
                continue
            q = torch.from_numpy(qall[:b]).cuda()
            out = g.alloc_outputs(b, topk, latents=bool(L))
            for _ in range(3):
                g.query_into(q, out, topk=topk)
            st, sc, fi = [], [], []
            for _ in range(a.steps):
                if a.flush != "none":
                    flush.fill_(1.0)
                if flush2 is not None:
                    flush2.sum()
                g.query_into(q, out, topk=topk)
                ev[3].synchronize()
                st.append(ev[0].elapsed_time(ev[3]))
                sc.append(ev[1].elapsed_time(ev[2]))
                fi.append(ev[2].elapsed_time(ev[3]))
            ms = statistics.median(st)
            scm = statistics.median(sc)
            rec = dict(scorer=scorer, n=n, b=b, topk=topk, flush=a.flush, step_ms=ms, score_ms=scm, finalize_ms=statistics.median(fi),
                       lookups_per_s=b / (ms / 1e3),
                       score_hbm_frac=n * 1540 / (scm / 1e3) / 1e9 / peaks["hbm_gbs"],
                       score_tensor_frac=2 * b * n * 768 / (scm / 1e3) / 1e12 / peaks["bf16_tflops"])
            print(json.dumps(rec), flush=True)
    g.set_profile_events(None)


if __name__ == "__main__":
    main()
