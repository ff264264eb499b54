"""Benchmark of the batched NIRVANA cache lookup (BASELINE.json metric) on B200.

python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4|c2|c3|c5|c1] [--batch B]
python bench.py --impl reference ...     (the fp64 CPU oracle, timed on the host cores)

One step = one full lookup batch: query ingest (normalise + bf16), exact cosine scan of every
cached entry with fused top-k, merge across scan splits (and across shards), Fig. 11 K map +
hole rule, latent gather of the hit states and LCBFU access counters.  Inputs are seeded,
synthetic, resident in HBM; L2 is flushed (a 512 MiB write) between timed steps and the step
time is taken with CUDA events on the launching stream, max over ranks.

Default workload: C4 (BASELINE.json configs[3]) -- one 10M-entry cache sharded over the N
GPUs, a 16,384-query global batch (16,384/N queries brought by each rank), strong scaling, so
that N = 1, 2, 4, 8 form one curve.  `--gpus N` without a torchrun environment re-launches
this script under torch.distributed.run with N ranks (one per GPU, rendezvous on 127.0.0.1).
`--config c2` is the 100K-entry single-GPU tensor-core workload (N > 1: independent replicas).
Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "cache lookups/sec (top-1+K+latent gather) at 1/2/4/8 B200; % of roofline"
UNIT = "lookups/s"
D = 768
L = 4 * 64 * 64 * 2
CONFIGS = {
    # BASELINE.json configs[1]: the headline single-GPU workload
    "c2": dict(n=100_000, b=4096, workload="C2: 100K cached entries x 768-d bf16, 4,096-query batches, "
                                          "K in {5,10,15,20,25}, 4x64x64 fp16 latents, 1 GPU (tensor-core path)"),
    # configs[2]: 1M entries, full per-K latent store, small batches (streaming/gather path)
    "c3": dict(n=1_000_000, b=32, workload="C3: 1M cached entries x 768-d bf16 with the full per-K 4x64x64 "
                                          "fp16 latent store (164 GB), batch 32"),
    # configs[0]: the small case the oracle finishes in seconds
    "c1": dict(n=1000, b=64, workload="C1: 1,000 entries x 768-d, 64 queries"),
    # configs[3]: 10M entries sharded across the N GPUs, 16K-query global batches (strong scaling)
    "c4": dict(n=10_000_000, b=16384, sharded=True,
               workload="C4: 10M cached entries x 768-d bf16 sharded across N B200, 16,384-query global batches, "
                        "top-1 merge across shards, K map, P2P latent fetch"),
    # configs[4]: 100M entries sharded across the N GPUs (the whole cache on one B200 at N = 1:
    # 154 GB of bf16 rows + 7 GB of metadata), Zipf-popular queries over entries, and every
    # round = one 16K-query lookup batch + LCBFU eviction of 1% of the live items + re-insertion
    # of as many fresh prompts as the eviction removed (strong scaling)
    "c5": dict(n=100_000_000, b=16384, sharded=True, maintenance=0.01, pool_slots=131_072,
               workload="C5: 100M cached entries x 768-d bf16 sharded across N B200, 16,384-query global "
                        "batches of Zipf-popular queries, LCBFU eviction of 1% of the live items + "
                        "re-insertion per round"),
}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """SM clock + clock-event-reason sampler during the timed region (B200_PROFILING.md clocks
    line): NVML polled every ~2 ms on a thread (a C2 timed region lasts only ~15 ms, shorter
    than nvidia-smi's start-up); nvidia-smi -lms 100 if NVML is unavailable."""

    _BITS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}

    def __init__(self, index: int):
        self.index, self.rows, self.proc, self.nv = index, [], None, None
        self.stop = threading.Event()

    def _nvml_handle(self):
        import pynvml
        import torch
        pynvml.nvmlInit()
        p = torch.cuda.get_device_properties(self.index)
        try:
            return pynvml.nvmlDeviceGetHandleByPciBusId(
                f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0".encode())
        except Exception:
            return pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def __enter__(self):
        try:
            import pynvml
            h = self._nvml_handle()
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            get_r = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
            first = threading.Event()

            def poll():
                while not self.stop.is_set():
                    self.rows.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), mx, get_r(h)))
                    first.set()
                    time.sleep(0.002)

            self.nv = threading.Thread(target=poll, daemon=True)
            self.nv.start()
            first.wait(timeout=1.0)   # the first sample precedes the timed region
            return self
        except Exception:
            self.nv = None
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.nv:
            self.stop.set()
            self.nv.join(timeout=1.0)
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        if self.nv is not None:
            sm = [float(r[0]) for r in self.rows]
            reasons = sorted({name for r in self.rows for bit, name in self._BITS.items() if r[2] & bit})
            return {"sm_mhz": statistics.median(sm), "sm_max_mhz": float(self.rows[0][1]), "reasons": reasons,
                    "samples": len(self.rows), "source": "nvml"}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows), "source": "nvidia-smi"}


def build_cache(B, torch, cfg, seed, dev):
    n = cfg["n"]
    emb, cl = __import__("synth").entries(n, seed=seed)
    import synth
    pres = synth.present_masks(n, seed=seed)
    # 2% entry headroom so the maintenance leg can re-insert after evicting 1% of the states
    g = B.NirvanaCache(entry_capacity=n + n // 50 + 64, latent_capacity=5 * n, dim=D, latent_bytes=L, device=dev)
    chunk = 8192
    for s in range(0, n, chunk):
        m = min(chunk, n - s)
        lat = synth.latents_torch(s, m, 5, L, seed=seed, device=f"cuda:{dev}")
        g.insert(torch.from_numpy(emb[s:s + m]).to(f"cuda:{dev}"), lat, present=pres[s:s + m])
        del lat
    return g, emb, cl, pres


def _host_threads():
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:
        return max(1, os.cpu_count() or 1)


def _oracle_queries_parallel(o, rows, nthreads):
    """The unchanged oracle, one query per call, on nthreads host threads: its C query is
    read-only on the cache with apply_counters=False and ctypes drops the GIL, so the calls
    run in parallel on the cores."""
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=nthreads) as ex:
        list(ex.map(lambda r: o.query(r[None, :], topk=1, want_latents=False, apply_counters=False), rows))


def cpu_baseline(emb, pres, q, budget_s=12.0, n_total=None):
    """Time the fp64 oracle (as it stands) on a bounded sample of the same workload: on one
    host thread, then on every host core (one query per thread at a time).  When emb is a
    slice of a larger cache (n_total rows; C4/C5), the scan cost is linear in the number of
    entries, so the rate over the slice is scaled by len(emb) / n_total to the full cache."""
    import oracle
    n_total = n_total or emb.shape[0]
    scale = emb.shape[0] / n_total
    o = oracle.OracleCache(dim=D, entry_capacity=emb.shape[0], latent_bytes=0)
    o.insert(emb, present=pres)
    done, t0 = 0, time.perf_counter()
    while done < q.shape[0] and time.perf_counter() - t0 < budget_s / 3:
        o.query(q[done:done + 1], topk=1, want_latents=False, apply_counters=False)
        done += 1
    dt1 = time.perf_counter() - t0
    v1 = done / dt1
    nt = _host_threads()
    # size the multi-core sample for ~2/3 of the budget from the single-thread rate
    m = int(min(q.shape[0], max(nt, v1 * nt * budget_s * 2 / 3)))
    t0 = time.perf_counter()
    _oracle_queries_parallel(o, q[:m], nt)
    dtn = time.perf_counter() - t0
    o.close()
    what = (f"the full {emb.shape[0]}-entry cache" if scale == 1 else
            f"the first {emb.shape[0]} entries of the {n_total}-entry cache, rate x {scale:.4g} "
            f"(the exhaustive scan is linear in the entry count)")
    return dict(value=m / dtn * scale, unit=UNIT, cores=nt, kind="oracle",
                sample=f"{m} queries of the same batch against {what} "
                       f"(fp64 scan + full sort + K map + holes; stored without latent payload bytes), "
                       f"{nt} host threads, {dtn:.1f} s",
                single_thread=dict(value=v1 * scale, cores=1, sample=f"{done} queries, {dt1:.1f} s"))


REF_SLICE = int(os.environ.get("REF_SLICE", "200000"))   # entries of a C4/C5 cache the oracle scans per sampled query (rate scaled)


def run_reference(args, cfg):
    """The reference arm: the fp64 oracle, unchanged, on the host cores (rank 0 only; other
    ranks exit without work).  Each step = one query per host thread of the workload's batch
    against the full cache (C1-C3) or against a REF_SLICE-entry slice of it with the rate
    scaled to the full cache (C4/C5: 10M-100M entries x 768 fp64 do not fit a bounded sample)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if rank != 0:
        return
    import synth
    n = cfg["n"]
    if cfg.get("sharded"):
        import torch
        ns = min(n, REF_SLICE)
        E = synth.TorchEntries(ns, seed=1000, device="cpu")
        emb = E.rows(torch.arange(ns, dtype=torch.int64)).numpy()
        pres = synth.present_masks(ns, seed=1000)
        q = E.queries(min(cfg["b"], 4096), qseed=1001)[0].numpy()
        scale = ns / n
        sample = (f"{{per_step}} queries per step against a {ns}-entry slice of the {n}-entry cache (same "
                  f"recipe), rate x {scale:.4g} (the exhaustive scan is linear in the entry count)")
    else:
        emb, cl = synth.entries(n, seed=1000)
        pres = synth.present_masks(n, seed=1000)
        q, _, _ = synth.queries(emb, cl, cfg["b"], seed=1001)
        scale = 1.0
        sample = f"{{per_step}} queries per step of the {cfg['b']}-query batch, full {n}-entry scan"
    import oracle
    o = oracle.OracleCache(dim=D, entry_capacity=emb.shape[0], latent_bytes=0)
    o.insert(emb, present=pres)
    nt = _host_threads()
    # one query per host thread per step (the oracle unchanged; see _oracle_queries_parallel)
    per_step = max(1, min(q.shape[0], int(os.environ.get("REF_QUERIES_PER_STEP", str(nt)))))
    for w in range(args.warmup):
        _oracle_queries_parallel(o, q[:per_step], nt)
    times, done = [], 0
    for s in range(args.steps):
        sel = q[(s * per_step) % q.shape[0]:][:per_step]
        t0 = time.perf_counter()
        _oracle_queries_parallel(o, sel, nt)
        times.append(time.perf_counter() - t0)
        done += len(sel)
    v = done / sum(times) * scale
    line = dict(impl="reference", metric=METRIC, value=v, unit=UNIT, n_gpus=world, steps=args.steps,
                warmup=args.warmup, ms_per_step=1e3 * statistics.mean(times), higher_is_better=True,
                scaling="strong" if cfg.get("sharded") else "weak", vs_baseline=None, dtype="f64", data="synthetic",
                config=dict(workload=cfg["workload"], entries=n, batch=cfg["b"], dim=D, latent_bytes=L, topk=1,
                            parallelism=f"{nt} host threads (fp64 oracle, one query per thread)"),
                cpu_baseline=dict(value=v, unit=UNIT, cores=nt, kind="oracle", sample=sample.format(per_step=per_step)),
                e2e=dict(value=v, unit=UNIT, h2d_bytes_per_step=0, d2h_bytes_per_step=0))
    print(json.dumps(line), flush=True)


def run_sharded(args, cfg):
    """C4: one cache of n entries sharded over the N ranks (strong scaling), global batch of
    B queries (B/N brought by each rank), latent states read through the declared aliased
    pool (the 10M x 5 x 32 KiB store does not fit HBM)."""
    import torch
    import torch.distributed as dist
    from paper_2312_04429_b200 import binding as B
    from paper_2312_04429_b200.sharded import ShardedCache, TorchComm
    import synth

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", str(_free_port()))
    os.environ.setdefault("RANK", "0")
    os.environ.setdefault("WORLD_SIZE", "1")
    if int(os.environ["WORLD_SIZE"]) > 1:
        # NCCL's communicator set-up lines (ranks, transports) go to the log (stderr), not stdout
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    comm = TorchComm()
    world, rank = comm.world, comm.rank
    n, b = cfg["n"], cfg["b"]
    bl = b // world
    pool_slots = cfg.get("pool_slots", 262_144)
    push = args.exchange == "push"
    maint = cfg.get("maintenance", 0.0)
    per_rank = (n + world - 1) // world
    # C5 re-inserts as many entries as each round's eviction removed: 0.5% entry headroom
    # absorbs the uneven per-rank split of dirty entries vs placement of the fresh ones
    sc = ShardedCache(comm, entry_capacity=per_rank + (per_rank // 200 if maint else 0) + 1024,
                      latent_capacity=pool_slots,
                      dim=D, latent_bytes=L, latent_alias=True, push_max_nb=bl if push else 0, push_max_topk=1)
    for s in range(0, pool_slots, 8192):
        m = min(8192, pool_slots - s)
        sc.cache.pool_write(s, synth.latents_torch(s, m, 1, L, seed=7, device="cuda").view(m, L))
    E = synth.TorchEntries(n, seed=1000, device="cuda")
    pres = synth.present_masks(n, seed=1000)
    chunk = 65536
    for s in range(0, n, chunk):
        m = min(chunk, n - s)
        rows = E.rows(torch.arange(s, s + m, dtype=torch.int64, device="cuda"))
        sc.insert(rows, None, present=pres[s:s + m])
    del rows
    q, _, _ = E.queries(bl, qseed=1001 + 7919 * rank)
    out = sc.alloc_outputs(bl, 1, latents=True)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(max(3, args.warmup)):
        sc.query_into(q, out)
    sc.cache.set_profile_events(ev)
    torch.cuda.synchronize()
    dist.barrier()
    step_ms, score_ms = [], []
    launches0 = sc.cache.kernel_launches
    next_row = n                 # fresh prompts of later rounds: rows n, n+1, ... of the same recipe
    m_ev, m_ins, m_items, m_dirty = [], [], [], []

    def maintenance_round():
        # a9 + a10 at C5: evict 1% of the live items (collective, exact global LCBFU selection
        # with the histograms reduced over peer memory), then insert as many fresh prompts as
        # the eviction removed whole (their states come from the aliased pool)
        nonlocal next_row
        live = comm.all_reduce_sum(torch.tensor([sc.cache.evict_units], dtype=torch.int64,
                                                device="cuda")).item()
        nev = max(1, int(live * maint))
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        _, nd = sc.evict(nev, lists=False)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        nd = comm.all_reduce_sum(torch.tensor([nd], dtype=torch.int64, device="cuda")).item()
        t_ins = 0.0
        for s0 in range(0, nd, 65536):
            m = min(65536, nd - s0)
            # the fresh prompts' embeddings are generated outside the timed insert call
            rows = E.rows(torch.arange(next_row + s0, next_row + s0 + m, dtype=torch.int64, device="cuda"))
            torch.cuda.synchronize()
            ta = time.perf_counter()
            sc.insert(rows, None)
            torch.cuda.synchronize()
            t_ins += time.perf_counter() - ta
        next_row += nd
        tt = torch.tensor([t1 - t0, t_ins], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        m_ev.append(1e3 * float(tt[0]))
        m_ins.append(1e3 * float(tt[1]))
        m_items.append(nev)
        m_dirty.append(nd)

    if maint:
        maintenance_round()      # warm-up round (lazy workspace allocations)
    with Clocks(torch.cuda.current_device()) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)
            dist.barrier()
            e0.record()
            sc.query_into(q, out)
            e1.record()
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            score_ms.append(ev[1].elapsed_time(ev[2]))
            if maint:
                maintenance_round()
    launches = sc.cache.kernel_launches - launches0
    sc.cache.set_profile_events(None)
    t = torch.tensor([sum(step_ms)], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tot = float(t.item())
    k_np = out["k"].cpu().numpy()
    # end to end through the public sharded API (ShardedCache.query_host): every step copies
    # this rank's fp32 query rows from pinned host memory, runs the collective lookup and reads
    # ids / scores / K / status back into pinned host memory; max over ranks of the wall time
    e2e = None
    if not args.no_e2e:
        qh = q.cpu().pin_memory()
        ho = dict(ids=torch.empty((bl, 1), dtype=torch.int64).pin_memory(),
                  scores=torch.empty((bl, 1), dtype=torch.float32).pin_memory(),
                  k=torch.empty(bl, dtype=torch.int32).pin_memory(),
                  status=torch.empty(bl, dtype=torch.int32).pin_memory())
        for _ in range(2):
            sc.query_host(qh, ho, out)
        e_ms = []
        for _ in range(args.steps):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            sc.query_host(qh, ho, out)
            e_ms.append(1e3 * (time.perf_counter() - t0))
        et = torch.tensor([sum(e_ms)], device="cuda", dtype=torch.float64)
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
        et = float(et.item())
        qd_raw = torch.empty_like(qh, device="cuda")
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        qd_raw.copy_(qh, non_blocking=True)
        torch.cuda.synchronize()
        h0.record()
        for _ in range(args.steps):
            qd_raw.copy_(qh, non_blocking=True)
        h1.record()
        torch.cuda.synchronize()
        h2d_ms = h0.elapsed_time(h1) / args.steps
        bound_ms = max(h2d_ms, tot / args.steps)
        if not maint:   # (C5's eviction rounds change the cache between the two measurements)
            assert np.array_equal(ho["k"].numpy(), k_np), "host-API lookup disagrees with the device-buffer lookup"
        e2e = dict(value=b * args.steps / (et / 1e3), unit=UNIT, h2d_bytes_per_step=b * D * 4,
                   d2h_bytes_per_step=b * (8 + 4 + 4 + 4), h2d_gbs=bl * D * 4 / (h2d_ms / 1e3) / 1e9,
                   bound=dict(ms=bound_ms, by="host-to-device copy" if h2d_ms > tot / args.steps else "device step",
                              frac=bound_ms / (et / args.steps)),
                   note="ShardedCache.query_host on every rank: fp32 queries from pinned host memory in, "
                        "ids/scores/K/status back to pinned host memory, latent states fetched into the "
                        "denoiser's device input buffer; wall clock, max over ranks")
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ns = min(n, REF_SLICE)
        emb_s = E.rows(torch.arange(ns, dtype=torch.int64, device="cuda")).cpu().numpy()
        cpu = cpu_baseline(emb_s, pres[:ns], q.cpu().numpy(), n_total=n)
        del emb_s
    hbm, tflops, peak_src = _peaks()
    try:
        tf_sus = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops_sustained"]
    except Exception:
        tf_sus = 1400.0
    n_local = sc.cache.stats()["live_entries"]
    sc_ms = statistics.mean(score_ms)
    flops = 2.0 * b * n_local * D
    ach = flops / (sc_ms / 1e3) / 1e12
    if rank == 0:
        line = dict(metric=METRIC, value=b * args.steps / (tot / 1e3), unit=UNIT, n_gpus=world, steps=args.steps,
                    warmup=args.warmup, ms_per_step=tot / args.steps, higher_is_better=True, scaling="strong",
                    vs_baseline=None, dtype="bf16",
                    data="synthetic on-device (counter-hash clustered unit-norm 768-d entries, Zipf anchors)",
                    config=dict(workload=cfg["workload"], entries=n, batch=b, dim=D, latent_bytes=L, topk=1,
                                scorer="tc",
                                parallelism=(f"entry-sharded x{world} (fused push exchange: ingest kernel stores "
                                             f"query rows and local-merge kernel stores 16-B records straight "
                                             f"into peer arenas over NVLink, epoch flags; P2P latent fetch)")
                                if push else (f"entry-sharded x{world} (NCCL all-gather of queries and 16-B "
                                              f"records, P2P latent fetch)"),
                                latent_pool=f"aliased, {pool_slots} slots per rank",
                                l2="flushed between timed steps (512 MiB write)", hit_rate=float((k_np > 0).mean())),
                    kernel_ms=dict(score_local=sc_ms),
                    roofline=dict(bound="tensor", achieved=ach, peak=tf_sus, unit="TFLOP/s", frac=ach / tf_sus,
                                  kernel="score_tc (rank 0 shard)",
                                  peak_source=peak_src + ", sustained bf16 (a ~0.2 s kernel runs under the "
                                                         "power cap)",
                                  traffic=_ncu_traffic("tc", f"{args.config}_n{world}") or _ncu_traffic("tc", args.config),
                                  algorithmic_per_launch=flops),
                    cpu_baseline=cpu, e2e=e2e, gpu_launches=launches, clocks=clk.summary())
        if maint:
            lk = tot / args.steps
            line["maintenance"] = dict(
                evict_items=m_items[1:], evict_ms=m_ev[1:], dirty_removed=m_dirty[1:], insert_entries=m_dirty[1:],
                insert_ms=m_ins[1:], round_ms=[lk + a + c for a, c in zip(m_ev[1:], m_ins[1:])],
                lookups_per_s_incl_maintenance=b * args.steps / ((tot + sum(m_ev[1:]) + sum(m_ins[1:])) / 1e3),
                note="per timed round, after the lookup: LCBFU eviction of 1% of the live items (N = 1: the "
                     "fused single-launch eviction; N > 1: 8 radix-select passes with the histograms summed "
                     "over peer memory, then apply + dirty-entry removal; host wall clock, max over ranks) and "
                     "the insertion of as many fresh prompts as it removed (normalise + slot allocation + "
                     "metadata; aliased latent pool); value counts the lookups only")
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def _free_port() -> int:
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def _spawn(args) -> int:
    """`--gpus N` without a torch.distributed environment: re-launch this script with N ranks
    (one process per GPU) under torch.distributed.run on 127.0.0.1; rank 0 prints the line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def run_dry(args):
    """Launcher / rendezvous / max-over-ranks check without a GPU (gloo): the same rank plumbing
    as the GPU runs, a barrier + tiny all-reduce as the "step"; rank 0 prints a line flagged
    dry_run with no throughput.  Used by the CPU tests of the spawner."""
    import torch
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", str(_free_port()))
    os.environ.setdefault("RANK", "0")
    os.environ.setdefault("WORLD_SIZE", "1")
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    for _ in range(args.warmup):
        dist.barrier()
    times = []
    for _ in range(args.steps):
        dist.barrier()
        t0 = time.perf_counter()
        x = torch.full((1,), float(rank))
        dist.all_reduce(x)
        times.append(time.perf_counter() - t0)
        assert x.item() == world * (world - 1) / 2
    t = torch.tensor([sum(times)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps(dict(dry_run=True, metric=METRIC, value=None, unit=UNIT, n_gpus=world, steps=args.steps,
                              warmup=args.warmup, ms_per_step=1e3 * float(t.item()) / max(1, args.steps),
                              note="launcher check only (gloo barrier + all-reduce per step, no GPU work)")),
              flush=True)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=list(CONFIGS))
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--scorer", default="auto", choices=["auto", "tc", "tc1", "stream"],
                    help="tc1 = single-CTA tensor-core scan (auto/tc use CTA pairs for > 128 queries)")
    ap.add_argument("--exchange", default="push", choices=["push", "nccl"],
                    help="sharded configs (c4, c5): fused P2P push exchange or NCCL all-gathers")
    ap.add_argument("--slices", type=int, default=0,
                    help="query slices of cache_query_batch (0 = library auto, 1 = one scan launch)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-maintenance", action="store_true")
    ap.add_argument("--dry-run", action="store_true", help="launcher check on CPU (gloo), no GPU work")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(_spawn(args))
    if "WORLD_SIZE" in os.environ and int(os.environ["WORLD_SIZE"]) != args.gpus:
        print(f"bench.py: WORLD_SIZE={os.environ['WORLD_SIZE']} overrides --gpus {args.gpus}", file=sys.stderr)
    cfg = dict(CONFIGS[args.config])
    if args.batch:
        cfg["b"] = args.batch
    if args.dry_run:
        return run_dry(args)
    if args.impl == "reference":
        return run_reference(args, cfg)
    if cfg.get("sharded"):
        return run_sharded(args, cfg)
    return run_single(args, cfg)


def run_single(args, cfg):
    """C1-C3 (and C2 replicas at N > 1): one cache per GPU."""
    import torch
    import torch.distributed as dist
    from paper_2312_04429_b200 import binding as B
    import synth

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = local
    g, emb, cl, pres = build_cache(B, torch, cfg, seed=1000, dev=dev)
    g.set_scorer({"auto": B.SCORER_AUTO, "tc": B.SCORER_TC, "tc1": B.SCORER_TC_SINGLE,
                  "stream": B.SCORER_STREAM}[args.scorer])
    g.set_query_slices(args.slices)
    b = cfg["b"]
    q_np, _, _ = synth.queries(emb, cl, b, seed=1001 + 7919 * rank)
    q = torch.from_numpy(q_np).cuda()
    out = g.alloc_outputs(b, 1, latents=True)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    g.set_profile_events(ev)
    for _ in range(max(3, args.warmup)):
        g.query_into(q, out)
    torch.cuda.synchronize()
    step_ms, score_ms, prep_ms, fin_ms = [], [], [], []
    launches0 = g.kernel_launches
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    # timed steps: two events on the launching stream around each whole lookup, no library-
    # internal events (they would sit between the kernels and break the programmatic-launch
    # overlap); the per-kernel split comes from a second pass with the library's events
    g.set_profile_events(None)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(torch.cuda.current_device()) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)
            e0.record(stream)
            g.query_into(q, out)
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
        torch.cuda.synchronize()
    launches = g.kernel_launches - launches0
    g.set_profile_events(ev)
    for _ in range(args.steps):
        flush.fill_(1.0)
        g.query_into(q, out)
        ev[3].synchronize()
        prep_ms.append(ev[0].elapsed_time(ev[1]))
        score_ms.append(ev[1].elapsed_time(ev[2]))
        fin_ms.append(ev[2].elapsed_time(ev[3]))
    torch.cuda.synchronize()
    g.set_profile_events(None)
    tot = sum(step_ms)
    if world > 1:
        t = torch.tensor([tot], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
        tot = float(t.item())
    value = b * world * args.steps / (tot / 1e3)
    k_np = out["k"].cpu().numpy()
    hbm, tflops, peak_src = _peaks()
    n = cfg["n"]
    sc_ms = statistics.mean(score_ms)
    scorer_used = "stream" if args.scorer == "stream" else "tc"
    flops = 2.0 * b * n * D
    bytes_scan = n * (2 * D + 4) + b * D * 2          # entry rows + inv-norms + the query tile
    # the binding resource: tensor if flops / peak_tensor > bytes / peak_hbm (C2), else HBM (C3)
    if scorer_used == "tc" and flops / (tflops * 1e12) >= bytes_scan / (hbm * 1e9):
        achieved = flops / (sc_ms / 1e3) / 1e12
        roof = dict(bound="tensor", achieved=achieved, peak=tflops, unit="TFLOP/s", frac=achieved / tflops)
    else:
        achieved = bytes_scan / (sc_ms / 1e3) / 1e9
        roof = dict(bound="hbm", achieved=achieved, peak=hbm, unit="GB/s", frac=achieved / hbm)
    roof["kernel"] = f"score_{scorer_used}"
    roof["peak_source"] = peak_src
    roof["traffic"] = _ncu_traffic(scorer_used, args.config)
    roof["algorithmic_per_launch"] = flops if roof["bound"] == "tensor" else bytes_scan
    # the gather (finalize) kernel is HBM-bound: 2 x 32 KiB per hit (pool read + denoiser-buffer
    # write) + the partial records it merges; reported beside the dominant kernel
    fin_ms = statistics.mean(fin_ms)
    # with query slices the events time the LAST slice's finalize (the earlier ones run on the
    # library's side stream under the next slice's scan): count that slice's rows and hits
    # (slice rule of cache_set_query_slices: slices of ceil(b / n) rounded up to 256 rows)
    ns = args.slices if args.slices > 0 else 1   # library auto = one launch
    if args.scorer == "tc1":
        ns = 1
    sub = -(-(-(-b // ns)) // 256) * 256 if ns > 1 else b
    last0 = ((b - 1) // sub) * sub if ns > 1 else 0
    hits = int((out["k"][last0:] > 0).sum().item())
    g_bytes = 2 * L * hits + (b - last0) * 16 * 64
    gather_roof = dict(bound="hbm", achieved=g_bytes / (fin_ms / 1e3) / 1e9, peak=hbm, unit="GB/s",
                       frac=g_bytes / (fin_ms / 1e3) / 1e9 / hbm, kernel="finalize_gather",
                       algorithmic_per_launch=g_bytes)
    # end-to-end through the public host-buffer API (H2D queries + D2H results incl. latents)
    e2e = None
    if not args.no_e2e:
        qh = torch.from_numpy(q_np).pin_memory()
        ho = dict(ids=torch.empty((b, 1), dtype=torch.int64).pin_memory(),
                  scores=torch.empty((b, 1), dtype=torch.float32).pin_memory(),
                  k=torch.empty(b, dtype=torch.int32).pin_memory(),
                  status=torch.empty(b, dtype=torch.int32).pin_memory(),
                  latents=torch.empty((b, L), dtype=torch.uint8, device="cuda"))   # the denoiser's input buffer
        for _ in range(3):
            g.query_host(qh, out=ho)
        e_ms = []
        for _ in range(args.steps):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            g.query_host(qh, out=ho)
            e_ms.append(1e3 * (time.perf_counter() - t0))
        et = sum(e_ms)
        if world > 1:
            t = torch.tensor([et], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            et = float(t.item())
        # the host link's own rate for the same bytes (a plain pinned copy of the query batch):
        # the end-to-end call cannot beat max(device step, this copy)
        qd_raw = torch.empty_like(qh, device="cuda")
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        qd_raw.copy_(qh, non_blocking=True)
        torch.cuda.synchronize()
        h0.record()
        for _ in range(args.steps):
            qd_raw.copy_(qh, non_blocking=True)
        h1.record()
        torch.cuda.synchronize()
        h2d_ms = h0.elapsed_time(h1) / args.steps
        bound_ms = max(h2d_ms, tot / args.steps)
        e2e_sync = dict(value=b * world * args.steps / (et / 1e3), bound_frac=bound_ms / (et / args.steps),
                        note="cache_query_batch_host (synchronous per call), L2 flushed before every call")
        # pipelined host calls (cache_query_submit / _complete, two slots): batch i+1's upload
        # overlaps batch i's lookup; every step still uploads its queries from pinned host memory
        # and reads its results back.  No flush inside the loop: the scan's inputs (154 MB of rows
        # + the 16.4 GB latent pool) exceed the 126 MB L2.
        qhs = [qh, qh.clone().pin_memory()]
        lats = [ho["latents"], torch.empty_like(ho["latents"])]
        outs = [ho, {k: (torch.empty_like(v).pin_memory() if k != "latents" else None) for k, v in ho.items()}]
        for sl in (0, 1):
            g.submit(sl, qhs[sl], 1, lats[sl])
        for sl in (0, 1):
            g.complete(sl, outs[sl])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        g.submit(0, qhs[0], 1, lats[0])
        for i in range(args.steps):
            if i + 1 < args.steps:
                g.submit((i + 1) % 2, qhs[(i + 1) % 2], 1, lats[(i + 1) % 2])
            g.complete(i % 2, outs[i % 2])
        ep = 1e3 * (time.perf_counter() - t0)
        if world > 1:
            t = torch.tensor([ep], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ep = float(t.item())
        e2e = dict(value=b * world * args.steps / (ep / 1e3), unit=UNIT, h2d_bytes_per_step=b * D * 4,
                   d2h_bytes_per_step=b * (8 + 4 + 4 + 4),
                   h2d_gbs=b * D * 4 / (h2d_ms / 1e3) / 1e9,
                   bound=dict(ms=bound_ms, by="host-to-device copy" if h2d_ms > tot / args.steps else "device step",
                              frac=bound_ms / (ep / args.steps)),
                   sync=e2e_sync,
                   note="cache_query_submit / cache_query_complete, two slots: fp32 queries from pinned host "
                        "memory in (copy stream), ids/scores/K/status back to pinned host memory, latent states "
                        "gathered into the denoiser's device input buffers; wall clock from the first submit to "
                        "the last complete")
    # cache maintenance (a9, a10): LCBFU eviction of 1% of the live items (C5's recipe) and the
    # re-insertion of as many fresh prompts (all 5 states each) as the freed pool slots hold
    maint = None
    if not args.no_maintenance:
        import synth as _s
        rounds = []
        for r in range(4):               # a warm-up round (workspace growth to this n), then three
                                         # timed rounds: single host-timed calls are noisy
            st = g.stats()
            nev = max(5, st["live_items"] // 100)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ev_ids, dirty = g.evict(nev, view=True)   # the serving loop reads the lists in place
            t_ev = time.perf_counter() - t0
            n_new = nev // 5
            new_emb, _ = _s.entries(n_new, seed=4242 + r)
            new_lat = _s.latents_torch(10_000_000 + r * n_new, n_new, 5, L, seed=4242, device="cuda")
            ne = torch.from_numpy(new_emb).cuda()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            g.insert(ne, new_lat)
            t_in = time.perf_counter() - t0
            del new_lat, ne
            if r > 0:
                rounds.append((nev, t_ev, len(dirty), n_new, t_in, st["entry_hwm"]))
        ev_ms = [1e3 * x[1] for x in rounds]
        in_ms = [1e3 * x[4] for x in rounds]
        nev, n_new = rounds[-1][0], rounds[-1][3]
        med_ev, med_in = statistics.median(ev_ms), statistics.median(in_ms)
        scan_bytes = rounds[-1][5] * (4 + 4 + 4 * 5)   # one full sweep of the slot columns (the window path)
        maint = dict(evict_items=nev, evict_ms=med_ev, evict_ms_rounds=ev_ms, evict_items_per_s=nev / (med_ev / 1e3),
                     dirty_removed=rounds[-1][2], evict_scan_gbs=scan_bytes / (med_ev / 1e3) / 1e9,
                     insert_entries=n_new, insert_ms=med_in, insert_ms_rounds=in_ms,
                     insert_states_per_s=5 * n_new / (med_in / 1e3),
                     note="host wall clock around the synchronous calls, median of 3 rounds after a warm-up round "
                          "(evict 1% of the live items, re-insert as many prompts with all 5 states); eviction = "
                          "one cooperative select + apply launch (a block sample estimates the cut, one full "
                          "sweep of the slot columns -- 28 B per slot -- histograms every key and compacts the "
                          "keys below the estimate, the selection and the apply finish on them; two sweeps if the "
                          "estimate misses) with the lists emitted sorted in the kernel + D2H of the lists + "
                          "host bookkeeping")
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(emb, pres, q_np)
    if rank == 0:
        line = dict(metric=METRIC, value=value, unit=UNIT, n_gpus=world, steps=args.steps, warmup=args.warmup,
                    ms_per_step=tot / args.steps, higher_is_better=True, scaling="weak", vs_baseline=None,
                    dtype="bf16", data="synthetic (seeded clustered unit-norm 768-d embeddings, Zipf queries, "
                                       "hash-stamped latents)",
                    config=dict(workload=cfg["workload"], entries=n, batch=b, dim=D, latent_bytes=L, topk=1,
                                scorer=scorer_used, l2="flushed between timed steps (512 MiB write)",
                                parallelism=f"replicas x{world}" if world > 1 else "single GPU",
                                hit_rate=float((k_np > 0).mean()), query_slices=ns),
                    kernel_ms=dict(ingest=statistics.mean(prep_ms), score=sc_ms, finalize_gather=fin_ms),
                    roofline=roof, roofline_gather=gather_roof, cpu_baseline=cpu, e2e=e2e, gpu_launches=launches,
                    clocks=clk.summary(),
                    maintenance=maint)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _ncu_traffic(scorer, config):
    """dram bytes per launch of the dominant kernel from the committed ncu --set full summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(f"{config}:{scorer}")
    except Exception:
        return None


if __name__ == "__main__":
    main()
