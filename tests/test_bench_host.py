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
