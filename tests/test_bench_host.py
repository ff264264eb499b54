"""Host-side pieces of bench.py that run without a GPU: the oracle baseline on every host core
(the unchanged oracle, one query per thread) must give the same answers as the serial oracle,
and the reference arm must print the contract's JSON line."""
import json
import os
import subprocess
import sys

import numpy as np

import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_parallel_oracle_calls_match_serial(oracle_mod):
    import bench
    n = 3000
    emb, cl = synth.entries(n, seed=71)
    pres = synth.present_masks(n, seed=71)
    q, _, _ = synth.queries(emb, cl, 64, seed=72)
    o = oracle_mod.OracleCache(dim=768, entry_capacity=n, latent_bytes=0)
    o.insert(emb, present=pres)
    serial = [o.query(q[i:i + 1], topk=1, want_latents=False, apply_counters=False) for i in range(64)]
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=8) as ex:
        par = list(ex.map(lambda r: o.query(r[None, :], topk=1, want_latents=False, apply_counters=False), q))
    for a, b in zip(serial, par):
        assert np.array_equal(a["ids"], b["ids"]) and np.array_equal(a["k"], b["k"])
        assert np.array_equal(a["raw"], b["raw"])
    bench._oracle_queries_parallel(o, q[:16], 4)   # the bench helper runs and leaves no counters
    o.close()
    rep = bench.cpu_baseline(emb, pres, q, budget_s=1.5)
    assert rep["kind"] == "oracle" and rep["cores"] == bench._host_threads() and rep["value"] > 0
    assert rep["single_thread"]["cores"] == 1


def test_reference_arm_prints_the_contract_line():
    env = dict(os.environ, REF_QUERIES_PER_STEP="2")
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "c1", "--steps", "2",
                          "--warmup", "1"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "lookups/s" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["e2e"]["h2d_bytes_per_step"] == 0


def _json_lines(stdout):
    return [json.loads(l) for l in stdout.splitlines() if l.startswith("{")]


def test_spawner_runs_n_ranks_and_rank0_prints_one_line():
    """`bench.py --gpus 2` with no torchrun environment re-launches itself under
    torch.distributed.run with two ranks (rendezvous on 127.0.0.1); the dry run exercises that
    launcher, the barrier and the max-over-ranks reduction with gloo, and only rank 0 prints."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_PORT")}
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--dry-run", "--steps", "3", "--warmup", "1"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = _json_lines(out.stdout)
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2 and lines[0]["dry_run"] and lines[0]["steps"] == 3


def test_reference_arm_c4_slice_under_two_ranks():
    """The default (C4) reference arm launched the driver's way for N = 2: rank 0 alone times the
    oracle on a slice of the 10M-entry cache (rate scaled to the full cache) and prints
    n_gpus = 2; rank 1 exits 0 without work."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_PORT")}
    env["REF_QUERIES_PER_STEP"] = "2"
    env["REF_SLICE"] = "20000"
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2", "--steps", "1",
                          "--warmup", "0"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = _json_lines(out.stdout)
    assert len(lines) == 1
    line = lines[0]
    assert line["impl"] == "reference" and line["n_gpus"] == 2 and line["config"]["entries"] == 10_000_000
    assert line["scaling"] == "strong" and line["value"] > 0 and "slice" in line["cpu_baseline"]["sample"]
