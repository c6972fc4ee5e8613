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
