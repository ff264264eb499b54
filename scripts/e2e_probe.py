"""Where the end-to-end host call's time goes: raw pinned H2D bandwidth for the query bytes,
the device-resident call, and the host call (C2 shapes).  Diagnostic only."""
import time

import numpy as np
import torch

import synth
from paper_2312_04429_b200 import binding as B


def ev_ms(fn, reps=20):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def wall_ms(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    t = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        t.append(1e3 * (time.perf_counter() - t0))
    return float(np.median(t)), float(np.min(t))


def main():
    b, n, D, L = 4096, 100_000, 768, 32768
    for mb in (1, 4, 12.6, 64):
        nb = int(mb * 2**20)
        h = torch.empty(nb, dtype=torch.uint8).pin_memory()
        d = torch.empty(nb, dtype=torch.uint8, device="cuda")
        ms = ev_ms(lambda: d.copy_(h, non_blocking=True))
        print(f"h2d {mb} MiB: {ms * 1e3:.1f} us = {nb / ms / 1e6:.1f} GB/s")
    g = B.NirvanaCache(entry_capacity=n, latent_capacity=5 * n, dim=D, latent_bytes=L)
    te = synth.TorchEntries(n, seed=1, device="cuda", dim=D)
    g.insert(te.rows(torch.arange(n, dtype=torch.int64, device="cuda")))
    qd = te.queries(b, qseed=2)[0].float().contiguous()
    out = g.alloc_outputs(b, 1, latents=False)
    print("device call ms", ev_ms(lambda: g.query_into(qd, out, topk=1)))
    qh = qd.cpu().pin_memory()
    ho = dict(ids=torch.empty((b, 1), dtype=torch.int64).pin_memory(),
              scores=torch.empty((b, 1), dtype=torch.float32).pin_memory(),
              k=torch.empty(b, dtype=torch.int32).pin_memory(), status=torch.empty(b, dtype=torch.int32).pin_memory(),
              latents=None)
    print("host call ms (median, min)", wall_ms(lambda: g.query_host(qh, out=ho)))


if __name__ == "__main__":
    main()
