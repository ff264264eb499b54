"""Experiment driver (not product): run the C2 lookup with a traced build of the scan and print
per-tile epilogue hold times and MMA accumulator waits of cluster 0 (exp_get_trace).

The traced build: `git apply scripts/exp_trace_instrumentation.diff` (clock64 stamps in the
CTA-pair kernel + an exp_get_trace export), `python -m paper_2312_04429_b200.build --force`,
run this on the GPU, then `git apply -R` and rebuild.  Results: profiles/r01_epilogue_trace.txt."""
import ctypes

import numpy as np
import torch

import synth
from paper_2312_04429_b200 import binding as B

n, b = 100_000, 4096
E = synth.TorchEntries(n, seed=1, device="cuda")
g = B.NirvanaCache(entry_capacity=n, latent_capacity=5 * n, dim=768, latent_bytes=0)
g.insert(E.rows(torch.arange(n, dtype=torch.int64, device="cuda")))
q = E.queries(b, qseed=2)[0]
out = g.alloc_outputs(b, 1, latents=False)
for _ in range(5):
    g.query_into(q, out, topk=1)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (4 * 256))()
B._lib.exp_get_trace(buf)
t = np.frombuffer(buf, dtype=np.uint64).reshape(4, 256).astype(np.int64)
ne = int((t[0] > 0).sum()); nm = int((t[2] > 0).sum())
hold = t[1, :ne] - t[0, :ne]
wait = t[3, :nm] - t[2, :nm]
tile = np.diff(t[0, :ne])
print("tiles traced", ne, nm)
print("epilogue hold (tfull seen -> release) cycles: median %d p90 %d max %d" % (np.median(hold), np.percentile(hold, 90), hold.max()))
print("tile period (tfull to tfull) cycles: median %d p90 %d" % (np.median(tile), np.percentile(tile, 90)))
print("MMA tempty wait cycles: median %d p90 %d max %d sum %d" % (np.median(wait), np.percentile(wait, 90), wait.max(), wait.sum()))
print("first 24 holds:", hold[:24].tolist())
print("first 24 waits:", wait[:24].tolist())
print("span cycles:", int(t[1, ne - 1] - t[2, 0]))
