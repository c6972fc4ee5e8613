"""-m "not gpu": bench.py's reference arm (the CPU oracle, this tier's reference)
prints one well-formed JSON line on the CPU, with the same config keys the GPU
arm reports."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0", "--rays-per-gpu", "20000"], capture_output=True, text=True, timeout=600,
                       cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "rays/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["steps"] == 1 and d["n_gpus"] == 1
    for k in ("workload", "n_triangles", "rays_per_gpu", "mode", "parallelism", "sample"):
        assert k in d["config"], k
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_arm_configs_match():
    sys.path.insert(0, ROOT)
    import argparse

    import bench
    args = argparse.Namespace(workload="sphere", rays_per_gpu=10_000_000, mode="boolean")
    c1 = bench.arm_config(args, 10_000, 1)
    c8 = bench.arm_config(args, 10_000, 8)
    assert c1["workload"] == c8["workload"] and "x8" in c8["parallelism"]


def test_parity_report_counts_mismatches_and_flags():
    """bench.py's parity block: an exact copy of the oracle's results is clean;
    a flipped boolean, a wrong count, a wrong nearest id and an out-of-tolerance
    point are each counted; flags are counted per category."""
    sys.path.insert(0, ROOT)
    import numpy as np

    import bench
    import oracle
    import synth
    V, T, S, E, _ = synth.workload("cube", 2000, seed=1)
    ref = oracle.run(V, T, S, E)
    got = {"hit": ref["hit"].copy(), "count": ref["count"].copy(), "tri": ref["tri"].copy(),
           "t": ref["t"].astype(np.float32), "dist": ref["dist"].astype(np.float32),
           "point": ref["point"].astype(np.float32)}
    r = bench.parity_report(got, ref, S, E, "cube")
    assert r["ok"] and r["rays"] == 2000 and r["mismatch_bool"] == r["mismatch_count"] == r["mismatch_tri"] == 0
    assert r["max_dt"] <= 1e-7 and r["flagged"]["any"] == int((ref["flags"] != 0).sum())
    hits = np.nonzero(ref["tri"] >= 0)[0]
    got["hit"][0] ^= 1
    got["count"][1] += 1
    got["tri"][hits[0]] = (got["tri"][hits[0]] + 1) % len(T)
    got["point"][hits[1]] += 1e-3
    r = bench.parity_report(got, ref, S, E, "cube")
    assert not r["ok"] and r["mismatch_bool"] == 1 and r["mismatch_count"] == 1 and r["mismatch_tri"] == 1
    assert r["tol_violations"] == 1
