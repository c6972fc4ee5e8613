#!/usr/bin/env python
"""Benchmark of the hot path: LBVH build + traversal/Moller-Trumbore (+ NCCL gather at N>1).

Contract: prints ONE JSON line on rank 0.

  step     = one pass of the whole hot path over one batch of synthetic input:
             rsi_rebuild (A1..A7: validate, extent, Morton, radix sort, Karras,
             refit/pack) + rsi_intersect (A8..A9) [+ NCCL gather of the per-ray
             outputs to rank 0 (A10) when N > 1].
  workload = closed UV-sphere mesh N_t = 10 000 (configs[1]/[2]), 1e7 segments
             per GPU with endpoints U[-1.5,1.5]^3 (weak scaling: each rank owns
             its own 1e7-ray slice), mode boolean (the north-star mode);
             barycentric and intercept_count rates are reported alongside.
  value    = total rays processed by all ranks / max-over-ranks device time.
  e2e      = the same metric through the C-ABI's rsi_test on pinned HOST
             buffers (H2D of mesh + rays, build, intersect, D2H of results).

`--impl reference` times the CPU oracle (the only reference this paper tier
has) on a bounded sample of the same workload.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = "rays/sec (boolean & barycentric) at N_t=1e4, N_r=1e7-1e8 on 1/2/4/8 B200"
UNIT = "rays/s"

# Algorithmic work model of the traversal kernel: SURVEY 8(d)'s per-unit
# figures (box tests and Moller-Trumbore tests per segment of the LBVH walk on
# each workload: any-hit for boolean, nearest for barycentric, all-hits for
# intercept_count) x 17 / 70 FP32 instructions per test.  The roofline's
# `achieved` is that fixed per-segment figure x the segments of one launch /
# the launch time -- a walk that needs fewer tests (a better tree) shows up as
# a higher fraction.  The tests per segment this build actually performs are
# MEASURED by an instrumented launch (RSI_OPT_COUNTERS) outside the timed
# region and reported next to it (`achieved_measured_work`).
WORK_MODEL = {
    "sphere": {"boolean": {"box_tests": 36.8, "mt_tests": 1.62},
               "barycentric": {"box_tests": 54.9, "mt_tests": 2.92},
               "intercept_count": {"box_tests": 69.3, "mt_tests": 3.97}},
    "terrain": {"boolean": {"box_tests": 37.8, "mt_tests": 1.50},
                "barycentric": {"box_tests": 43.7, "mt_tests": 1.94},
                "intercept_count": {"box_tests": 50.3, "mt_tests": 2.19}},
    "sphere1m": {"boolean": {"box_tests": 51.3, "mt_tests": 1.50},
                 "barycentric": {"box_tests": 78.8, "mt_tests": 2.83},
                 "intercept_count": {"box_tests": 103.2, "mt_tests": 3.99}},
}
WORK_MODEL["paper_terrain"] = {"boolean": {"box_tests": 46.3, "mt_tests": 1.50}}
FP32_PER_BOX = 17.0
FP32_PER_MT = 70.0
N_SM = 148
FP32_LANES = 128


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    # 1.25e7 per GPU: --gpus 8 is exactly the north-star row N_t = 1e4, N_r = 1e8
    ap.add_argument("--rays-per-gpu", type=int, default=12_500_000)
    ap.add_argument("--workload", default="sphere", choices=["sphere", "terrain", "paper_terrain", "sphere1m"])
    ap.add_argument("--mode", default="boolean", choices=["boolean", "barycentric", "intercept_count"])
    ap.add_argument("--no-extra-modes", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the other BASELINE configs (rank 0, N=1 only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the sphere1m parity sample (rank 0, N=1)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=0, help="oracle sample rays (0 = auto ~15 s)")
    ap.add_argument("--no-overlap", dest="overlap", action="store_false",
                    help="time the steps back to back on one stream and one handle (no step overlap)")
    ap.add_argument("--fused-gather", action="store_true",
                    help="N > 1: traversal writes straight into rank 0's buffers over NVLink (PeerOutputs) "
                         "instead of the pipelined NCCL gather")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        try:
            p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                  "-i", str(self.index), "-lms", "20"], stdout=subprocess.PIPE, text=True)
        except OSError:
            return
        while not self._stop.is_set():
            line = p.stdout.readline()
            if not line:
                break
            self.rows.append([x.strip() for x in line.split(",")])
        p.terminate()

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=3)

    def summary(self):
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows if len(r) >= 9 for k in range(4) if r[5 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


# ------------------------------------------------------------------ helpers
def workload_inputs(name: str, n: int, rank: int):
    seed = {"cube": 1, "sphere": 3, "terrain": 4, "paper_terrain": 6, "sphere1m": 5}[name] + 1000 * rank
    V, T, S, E, _ = synth.workload(name, n, seed=seed)
    return V, T, S, E


def host_cores() -> int:
    """Host cores this process may run on (the oracle's thread count)."""
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:
        return max(1, os.cpu_count() or 1)


def cpu_baseline(V, T, S, E, target_s=20.0, sample=0):
    """The oracle (as it stands, with its ambiguity flags) on a bounded sample
    of the same workload.  Returns (cpu_baseline dict, oracle results on the
    sample) -- the results feed the parity report."""
    import oracle
    cores = host_cores()
    if sample <= 0:
        # calibrate with a small run, then size for ~target_s of CPU work
        n0 = 200
        oracle.run(V, T, S[:n0], E[:n0], threads=cores)  # thread pool start-up outside the calibration
        t = time.perf_counter()
        oracle.run(V, T, S[:n0], E[:n0], threads=cores)
        dt = max(time.perf_counter() - t, 1e-3)
        sample = int(min(len(S), max(n0, n0 * target_s / dt)))
    t = time.perf_counter()
    ref = oracle.run(V, T, S[:sample], E[:sample], threads=cores)
    dt = time.perf_counter() - t
    return ({"value": sample / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
             "sample": f"first {sample} rays of the workload x all {len(T)} triangles, all modes + ambiguity "
                       f"flags at once (exhaustive fp64, {dt:.1f} s)"}, ref)


def parity_report(got: dict, ref: dict, S, E, label: str) -> dict:
    """GPU outputs of all three modes vs the oracle on the same rays, every ray
    (north_star agreement: boolean / intercept_count / nearest id exact on
    every ray -- flagged ones included and counted, never excused; t, dist,
    point within 1e-5, 1e-5 |d|, 1e-5 max(|O|, |E|)).  Flags: E edge/vertex,
    T endpoint touch, P near-parallel, B nearest tie, D dedup ambiguity."""
    import oracle
    fl = ref["flags"]
    m = ref["tri"] >= 0
    d = E.astype(np.float64) - S
    dn = np.maximum(np.linalg.norm(d, axis=1), 1e-30)
    scale = np.maximum(np.maximum(np.abs(S).max(1), np.abs(E).max(1)), 1e-30)
    both = m & (got["tri"] == ref["tri"])
    dt = np.abs(got["t"][both] - ref["t"][both])
    dd = np.abs(got["dist"][both] - ref["dist"][both]) / dn[both]
    dp = np.abs(got["point"][both] - ref["point"][both]).max(1) / scale[both]
    bad = ((got["hit"] != ref["hit"]) | (got["count"] != ref["count"]) | (got["tri"] != ref["tri"]))
    tol = np.zeros(len(S), bool)
    tol[np.nonzero(both)[0]] = (dt > 1e-5) | (dd > 1e-5) | (dp > 1e-5)
    names = {"E": oracle.FLAG_E, "T": oracle.FLAG_T, "P": oracle.FLAG_P, "B": oracle.FLAG_B, "D": oracle.FLAG_D}
    return {"workload": label, "rays": int(len(S)),
            "mismatch_bool": int((got["hit"] != ref["hit"]).sum()),
            "mismatch_count": int((got["count"] != ref["count"]).sum()),
            "mismatch_tri": int((got["tri"] != ref["tri"]).sum()),
            "tol_violations": int(tol.sum()),
            "max_dt": float(dt.max()) if dt.size else 0.0,
            "max_ddist_rel": float(dd.max()) if dd.size else 0.0,
            "max_dpoint_rel": float(dp.max()) if dp.size else 0.0,
            "flagged": {**{k: int(((fl & b) != 0).sum()) for k, b in names.items()}, "any": int((fl != 0).sum())},
            "flagged_mismatch": int((bad & (fl != 0)).sum()),
            "ok": bool(not bad.any() and not tol.any())}


def _traffic(mode: str, rays: int):
    """DRAM bytes per launch from the committed ncu capture of the same
    workload and ray count (profiles/traffic.json), if present."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        return int(t[mode]) if rays == int(t.get("rays", 10_000_000)) else None
    except (OSError, KeyError, ValueError):
        return None


def _ncu_traversal(mode: str):
    """Issue-slot use, SIMT width and cache hit rates of the traversal kernel from
    the committed ncu --set full capture (profiles/ncu_traversal.json): why the
    ALU fraction is what it is."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "ncu_traversal.json")))[mode]
    except (OSError, KeyError, ValueError):
        return None


def roofline(mode: str, rays: int, kernel_ms: float, sm_mhz: float | None, work: dict | None = None,
             workload: str = "sphere"):
    w = WORK_MODEL.get(workload, {}).get(mode) or WORK_MODEL["sphere"][mode]
    inst_per_ray = w["box_tests"] * FP32_PER_BOX + w["mt_tests"] * FP32_PER_MT
    clock = (sm_mhz or 1965.0) * 1e6
    peak = N_SM * FP32_LANES * clock / 1e12            # T FP32 inst/s (nominal: no measured FP32 peak)
    achieved = inst_per_ray * rays / (kernel_ms * 1e-3) / 1e12
    out = {"bound": "alu", "achieved": round(achieved, 4), "peak": round(peak, 4), "unit": "TFP32-inst/s",
           "frac": round(achieved / peak, 5), "traffic": _traffic(mode, rays),
           "traffic_unit": "DRAM bytes/launch (ncu); algorithmic = 24 B in + 1 / 4 / 24 B out per ray "
                           "(boolean / intercept_count / barycentric)",
           "kernel": f"k_trace<{mode}>", "kernel_ms": round(kernel_ms, 4), "ncu": _ncu_traversal(mode),
           "model": f"SURVEY 8(d) per-unit figure ({workload}, {mode}): {w['box_tests']:.1f} box x "
                    f"{FP32_PER_BOX:.0f} + {w['mt_tests']:.2f} MT x {FP32_PER_MT:.0f} = {inst_per_ray:.0f} "
                    "FP32 inst/ray; peak = nominal 148 SM x 128 FP32 lanes x median sm_mhz"}
    if work:
        mi = work["box_tests"] * FP32_PER_BOX + work["mt_tests"] * FP32_PER_MT
        out["achieved_measured_work"] = round(mi * rays / (kernel_ms * 1e-3) / 1e12, 4)
        out["frac_measured_work"] = round(mi * rays / (kernel_ms * 1e-3) / 1e12 / peak, 5)
        out["measured_work"] = (f"{work['box_tests']:.2f} box + {work['mt_tests']:.2f} MT per ray measured "
                                f"(RSI_OPT_COUNTERS) = {mi:.0f} FP32 inst/ray")
    return out


def oracle_run(V, T, S, E):
    import oracle
    return oracle.run(V, T, S, E)


def gpu_outputs(h, Sd, Ed) -> dict:
    """All three modes through rsi_intersect on the given handle, as host numpy."""
    from paper_2305_01867_b200 import rsi
    got = {"hit": rsi.rsi_intersect(h, Sd, Ed, "boolean")["hit"].cpu().numpy(),
           "count": rsi.rsi_intersect(h, Sd, Ed, "intercept_count")["count"].cpu().numpy()}
    got.update({k: v.cpu().numpy() for k, v in rsi.rsi_intersect(h, Sd, Ed, "barycentric").items()})
    return got


def pcie_link(index: int) -> str | None:
    try:
        r = subprocess.run(["nvidia-smi", "--query-gpu=pcie.link.gen.current,pcie.link.gen.max,"
                            "pcie.link.width.current,pcie.link.width.max", "--format=csv,noheader",
                            "-i", str(index)], capture_output=True, text=True, timeout=20)
        g, gm, w, wm = [x.strip() for x in r.stdout.strip().split(",")]
        return f"PCIe gen {g} (max {gm}) x{w} (max x{wm})"
    except Exception:  # noqa: BLE001
        return None


def pcie_ceiling(dev, ray_bytes: int, d2h_bytes: int, reps: int = 5) -> dict:
    """The host->device ceiling of the e2e path, measured the ways the path can
    copy: the step's ray bytes (2 arrays) as one copy per array, in 1 Mi-ray
    chunks on one stream, and in 1 Mi-ray chunks alternating two streams
    (rsi_test's pipeline), each timed with CUDA events, best of `reps`.  The
    fastest is the ceiling (the largest achievable GB/s; rsi_test cannot move
    its inputs faster).  The D2H of the outputs (other direction) and the
    last chunk's traversal; mesh and output copies are not counted, so the
    ceiling is a lower bound on any e2e step time)."""
    import torch
    nb = 2 * ray_bytes
    hb = torch.empty(nb, dtype=torch.uint8).pin_memory()
    db = torch.empty(nb, dtype=torch.uint8, device=dev)
    chunk = (1 << 20) * 12
    streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
    cur = torch.cuda.current_stream(dev)

    def run(kind):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cur)
        if kind == "single":
            for half in (0, ray_bytes):
                db[half:half + ray_bytes].copy_(hb[half:half + ray_bytes], non_blocking=True)
        else:
            for st in streams:
                st.wait_event(a)
            k = 0
            for half in (0, ray_bytes):
                for o in range(0, ray_bytes, chunk):
                    e = min(o + chunk, ray_bytes)
                    st = streams[k % 2] if kind == "chunk2" else streams[0]
                    with torch.cuda.stream(st):
                        db[half + o:half + e].copy_(hb[half + o:half + e], non_blocking=True)
                    k += 1
            for st in streams:
                cur.wait_stream(st)
        b.record(cur)
        torch.cuda.synchronize(dev)
        return a.elapsed_time(b)

    best = {}
    for kind in ("single", "chunk1", "chunk2"):
        run(kind)
        best[kind] = min(run(kind) for _ in range(reps))
    del hb, db
    kind = min(best, key=best.get)
    return {"ms": best[kind], "h2d_GBps": nb / best[kind] / 1e6, "method": kind,
            "candidates_ms": {k: round(v, 4) for k, v in best.items()}, "link": pcie_link(dev.index or 0)}


# ------------------------------------------------------------------ reference arm
def arm_config(args, n_tri: int, world: int, backend: str = "nccl") -> dict:
    """The `config` both arms report (the reference arm adds its sample)."""
    return {"workload": f"{args.workload} N_t={n_tri}, N_r={args.rays_per_gpu}/GPU, mode={args.mode}",
            "n_triangles": n_tri, "rays_per_gpu": args.rays_per_gpu, "mode": args.mode,
            "parallelism": f"ray-sharded x{world}" + ((" + fused NVLink writes to rank 0" if getattr(args, "fused_gather", False)
                                                     else f" + {backend} gather to rank 0") if world > 1 else ""),
            "l2": f"inputs larger than L2 ({args.rays_per_gpu * 24 / 1e6:.0f} MB of segments per GPU; no flush)",
            "step": "rsi_rebuild + rsi_intersect" + (" + gather" if world > 1 else "")
                    + " (RSI_OPT_DEFERRED_STATUS: build checks read back after the timed region)"
                    + ("; consecutive steps overlapped on two streams and two handles"
                       if getattr(args, "overlap", False) else "")}


def run_reference(args, rank: int, world: int):
    """The reference arm for this tier: the CPU oracle as it stands (exhaustive
    fp64 over all triangles), on the host cores, each step a bounded sample of
    the same workload; rank 0 only."""
    if rank != 0:
        return
    V, T, S, E = workload_inputs(args.workload, max(args.rays_per_gpu // 5, 20000), 0)
    import oracle
    # every host core this process may use: torchrun sets OMP_NUM_THREADS=1 per
    # rank, but rank 0 is the only one working here
    cores = host_cores()
    n0 = 100
    oracle.run(V, T, S[:n0], E[:n0], threads=cores)  # thread pool start-up outside the calibration
    t = time.perf_counter()
    oracle.run(V, T, S[:n0], E[:n0], threads=cores)
    dt = max(time.perf_counter() - t, 1e-3)
    per_step = int(max(n0, min(len(S), n0 * 4.0 / dt)))   # ~4 s of CPU per step
    for i in range(args.warmup):
        oracle.run(V, T, S[:per_step], E[:per_step], threads=cores)
    t = time.perf_counter()
    for i in range(args.steps):
        oracle.run(V, T, S[:per_step], E[:per_step], threads=cores)
    el = time.perf_counter() - t
    value = per_step * args.steps / el
    sample = (f"first {per_step} rays of the workload per step x all {len(T)} triangles, "
              f"exhaustive fp64, all modes + ambiguity flags at once")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded UV-sphere mesh, uniform segments; see DESIGN.md 4)",
            "config": {**arm_config(args, len(T), world), "sample": sample},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    from paper_2305_01867_b200 import rsi
    from paper_2305_01867_b200.sharded import FIELDS, GatherPipeline, PeerOutputs

    # one process per GPU; RSI_BENCH_BACKEND=gloo + more ranks than GPUs is a
    # launch/gather dry run on a single device (testing only, never a number)
    ndev = torch.cuda.device_count()
    torch.cuda.set_device(local % ndev)
    dev = torch.device("cuda", local % ndev)
    backend = os.environ.get("RSI_BENCH_BACKEND", "nccl")
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    n = args.rays_per_gpu
    V, T, S, E = workload_inputs(args.workload, n, rank)
    Vd, Td = torch.from_numpy(V).to(dev), torch.from_numpy(T).to(dev)
    Sd, Ed = torch.from_numpy(S).to(dev), torch.from_numpy(E).to(dev)
    stream = torch.cuda.current_stream(dev)
    # deferred build status: each step enqueues rebuild + intersect with no host
    # read-back in between (the device-side input checks still run every step;
    # their result is read once after the timed region)
    h = rsi.rsi_build(Vd, Td, rsi.Options(deferred_status=True))

    # a second handle for the overlapped steps (below); built once, rebuilt every step
    h_b = rsi.rsi_build(Vd, Td, rsi.Options(deferred_status=True)) if args.overlap else None

    last_out = {}

    def timed(mode: str, steps: int, warmup: int, clocks: bool, overlap: bool = False):
        # N > 1: the gather of step k (NCCL, its own stream) overlaps the build +
        # traversal of step k+1; two output slots, each reused only after its
        # previous gather completed (a device-side wait); all gathers finish
        # inside the timed region (drain before the end event).
        # overlap: consecutive steps alternate between two handles and two
        # streams, so step k+1's rebuild (small latency-bound grids) fills the
        # SMs that step k's persistent traversal frees in its tail, and step
        # k+1's traversal starts as soon as its own BVH is ready.  Every step
        # still does the whole rebuild + intersect; step k+2 reuses step k's
        # handle and outputs only after step k finished (same stream).
        peer = PeerOutputs(n * world, mode, dev) if (world > 1 and args.fused_gather) else None
        overlap = overlap and peer is None
        hs = [h, h_b] if overlap else [h]
        sts = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)] if overlap else [stream]
        if peer is not None:
            outs = [peer.outputs()]
            pipe = None
        else:
            outs = [rsi.alloc_outputs(n, mode, dev) for _ in range(2 if (world > 1 or overlap) else 1)]
            pipe = GatherPipeline(slots=2) if world > 1 else None

        def step(k, ev=None):
            out = outs[k % len(outs)]
            st = sts[k % len(sts)]
            hk = hs[k % len(hs)]
            with torch.cuda.stream(st):
                if pipe is not None and pipe.slots[k % 2] is not None:
                    pipe.slots[k % 2].wait()  # this slot's send buffer is free again
                if peer is not None:
                    peer.begin()  # rank 0 is done with the previous step's rows
                if ev is not None:
                    ev[0].record(st)
                rsi.rsi_rebuild(hk, Vd, Td)
                if ev is not None:
                    ev[1].record(st)
                rsi.rsi_intersect(hk, Sd, Ed, mode, out=out)
                if ev is not None:
                    ev[2].record(st)
                if pipe is not None:
                    pipe.start(k % 2, {f: out[f] for f in FIELDS[mode]}, n * world)
                if peer is not None:
                    peer.complete()  # device-side barrier: rank 0 holds every rank's rows

        for k in range(warmup):
            step(k)
        if pipe is not None:
            pipe.drain()
        torch.cuda.synchronize(dev)
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        sampler = ClockSampler(local) if clocks else None
        if sampler:
            sampler.__enter__()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        launches0 = rsi.rsi_launch_count()
        t0.record(stream)
        for st in sts:
            st.wait_stream(stream)
        for k in range(steps):
            step(k, None if overlap else evs[k])
        with torch.cuda.stream(sts[(steps - 1) % len(sts)]):
            if pipe is not None:
                pipe.drain()  # every step's outputs are on rank 0 before the end event
        for st in sts:
            stream.wait_stream(st)
        t1.record(stream)
        launches = rsi.rsi_launch_count() - launches0
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        if sampler:
            sampler.__exit__()
        ms = t0.elapsed_time(t1)
        # per-step build / query times only from the serial (non-overlapped) run:
        # overlapped events would include waits for the other stream's SMs
        build_ms = None if overlap else statistics.mean(e[0].elapsed_time(e[1]) for e in evs)
        query_ms = None if overlap else statistics.mean(e[1].elapsed_time(e[2]) for e in evs)
        if world > 1:
            tm = torch.tensor([ms, build_ms or 0.0, query_ms or 0.0], dtype=torch.float64, device=dev)
            dist.all_reduce(tm, op=dist.ReduceOp.MAX)
            ms = tm[0].item()
            if not overlap:
                build_ms, query_ms = tm[1].item(), tm[2].item()
        if world == 1 or peer is None:  # the last timed step's outputs (parity block below)
            last_out[mode] = outs[(steps - 1) % len(outs)]
        return ms, build_ms, query_ms, (sampler.summary() if sampler else None), launches

    def timed_pair(mode: str, steps: int, warmup: int, clocks: bool):
        """The serial run (per-step build / query events: the roofline's kernel
        time) and, with --overlap, the overlapped run that gives the value."""
        s_ms, build_ms, query_ms, s_clk, s_launch = timed(mode, steps, warmup, clocks and not args.overlap)
        if not args.overlap:
            return s_ms, build_ms, query_ms, s_clk, s_launch, None
        ms, _, _, clk, launches = timed(mode, steps, warmup, clocks, overlap=True)
        return ms, build_ms, query_ms, clk, launches, {"serial_ms_per_step": s_ms / steps,
                                                      "serial_value": n * world * steps / (s_ms * 1e-3)}

    ms, build_ms, query_ms, clk, launches, serial = timed_pair(args.mode, args.steps, max(args.warmup, 3), True)
    total_rays = n * world * args.steps
    value = total_rays / (ms * 1e-3)
    extra = {}
    if not args.no_extra_modes:
        for m in ("barycentric", "intercept_count"):
            if m == args.mode:
                continue
            mms, mb, mq, _, _, mser = timed_pair(m, args.steps, 3, False)
            extra[m] = {"value": n * world * args.steps / (mms * 1e-3), "ms_per_step": mms / args.steps,
                        "build_ms": mb, "query_ms": mq, "serial": mser}
    rsi.rsi_build_status(h)  # raises if any timed build failed its input checks
    if h_b is not None:
        rsi.rsi_build_status(h_b)
        h_b.free()
    stats = rsi.rsi_get_stats(h)

    # the other BASELINE.json configs (parity-test workloads), timed on this GPU
    # for context: rays/s of rebuild + intersect per step, 3 warm-up + 10 timed steps
    other = {}
    if world == 1 and not args.no_configs:
        def one_config(name, mode, n_rays):
            V2, T2, S2, E2 = workload_inputs(name, n_rays, 0)
            V2d, T2d = torch.from_numpy(V2).to(dev), torch.from_numpy(T2).to(dev)
            S2d, E2d = torch.from_numpy(S2).to(dev), torch.from_numpy(E2).to(dev)
            # same step as the headline: rebuild + intersect, consecutive steps
            # overlapped on two handles / streams unless --no-overlap
            nh = 2 if args.overlap else 1
            reps = 10  # timed steps (3 warm-ups)
            o2 = [rsi.alloc_outputs(n_rays, mode, dev) for _ in range(nh)]
            h2 = [rsi.rsi_build(V2d, T2d, rsi.Options(deferred_status=True)) for _ in range(nh)]
            st2 = [torch.cuda.Stream(dev) for _ in range(nh)] if args.overlap else [stream]

            def run(k):
                with torch.cuda.stream(st2[k % nh]):
                    rsi.rsi_rebuild(h2[k % nh], V2d, T2d)
                    rsi.rsi_intersect(h2[k % nh], S2d, E2d, mode, out=o2[k % nh])
            for k in range(3):
                run(k)
            torch.cuda.synchronize(dev)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for st in st2:
                st.wait_stream(stream)
            for k in range(reps):
                run(k)
            for st in st2:
                stream.wait_stream(st)
            b.record(stream)
            torch.cuda.synchronize(dev)
            ms3 = a.elapsed_time(b) / reps
            for hh in h2:
                rsi.rsi_build_status(hh)
                hh.free()
            return {"workload": f"{name} N_t={len(T2)}, N_r={n_rays}, {mode}", "value": n_rays / (ms3 * 1e-3),
                    "unit": UNIT, "ms_per_step": ms3}
        other["configs[0] cube all modes"] = [one_config("cube", m, 10_000)
                                              for m in ("boolean", "barycentric", "intercept_count")]
        other["configs[1] sphere 1e6 boolean"] = one_config("sphere", "boolean", 1_000_000)
        other["configs[3] folded terrain 1e7 intercept_count"] = one_config("terrain", "intercept_count", 10_000_000)
        other["paper-shaped terrain (P:148) 1e7 boolean"] = one_config("paper_terrain", "boolean", 10_000_000)
        other["configs[4] per-GPU share: sphere N_t=1e6, 1.25e7 boolean"] = one_config("sphere1m", "boolean",
                                                                                      12_500_000)
    # measured algorithmic work per ray (instrumented launch, outside the timed region)
    work = None
    with rsi.rsi_build(Vd, Td, rsi.Options(counters=True)) as hc:
        rsi.rsi_intersect(hc, Sd, Ed, args.mode)
        cs = rsi.rsi_get_stats(hc)
        work = {"box_tests": cs["box_tests"] / n, "mt_tests": cs["mt_tests"] / n}

    # e2e: through the C-ABI rsi_test on pinned host buffers (rank-local)
    e2e = None
    if not args.no_e2e:
        pin = lambda a: torch.from_numpy(a).pin_memory()  # noqa: E731
        hV, hT, hS, hE = pin(V), pin(T), pin(S), pin(E)
        hout = {k: v.pin_memory() for k, v in rsi.alloc_outputs(n, args.mode, "cpu").items()}
        for _ in range(2):
            rsi.rsi_test(hV, hT, hS, hE, {"mode": args.mode}, out=hout, sparse=False)
        e_steps = max(2, min(args.steps, 5))
        if world > 1:
            dist.barrier()
        t = time.perf_counter()
        for _ in range(e_steps):
            rsi.rsi_test(hV, hT, hS, hE, {"mode": args.mode}, out=hout, sparse=False)
        el = time.perf_counter() - t
        if world > 1:
            tt = torch.tensor([el], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            el = tt.item()
        h2d = V.nbytes + T.nbytes + S.nbytes + E.nbytes
        d2h = sum(v.numel() * v.element_size() for v in hout.values())
        e_ms = el / e_steps * 1e3
        ceil = pcie_ceiling(dev, S.nbytes, d2h)
        e2e = {"value": n * world * e_steps / el, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": e_ms,
               "api": "rsi_test (C-ABI, pinned host buffers, dense per-ray outputs)",
               "roofline": {"bound": "pcie_h2d", "ceiling_ms": ceil["ms"], "h2d_GBps": ceil["h2d_GBps"],
                            "frac": ceil["ms"] / e_ms, "link": ceil["link"], "method": ceil["method"],
                            "candidates_ms": ceil["candidates_ms"]}}
        del hV, hT, hS, hE, hout

    # the paper's own headline workload, end to end like its timings (P:144,
    # P:147-154): 1e7 rays against the 29 260-triangle terrain, host buffers in,
    # results out, through the C-ABI rsi_test (rank 0, N = 1 only; context)
    paper = None
    if rank == 0 and world == 1 and not args.no_configs and not args.no_e2e:
        Vp, Tp, Sp, Ep = workload_inputs("paper_terrain", 10_000_000, 0)
        pin = lambda a: torch.from_numpy(a).pin_memory()  # noqa: E731
        hVp, hTp, hSp, hEp = pin(Vp), pin(Tp), pin(Sp), pin(Ep)
        # the paper's best end-to-end time per mode (unstated GPU)
        paper_ms = {"boolean": (300.166, "original CUDA, P:152"),
                    "barycentric": (456.346, "PyCUDA with GPU post-processing (points, distances), P:184"),
                    "intercept_count": (334.192, "original CUDA, P:154")}
        paper = {"workload": f"paper_terrain N_t={len(Tp)}, N_r=10000000, e2e via rsi_test (pinned host buffers)"}
        for m, (pms, src) in paper_ms.items():
            nr = len(Sp)
            hout = rsi.alloc_outputs(nr, m, "cpu")
            hout = {k: v.pin_memory() for k, v in hout.items()}
            rsi.rsi_test(hVp, hTp, hSp, hEp, {"mode": m}, out=hout, sparse=False)
            reps = 3
            t = time.perf_counter()
            for _ in range(reps):  # dense per-ray outputs in pinned host memory (no host post-processing)
                rsi.rsi_test(hVp, hTp, hSp, hEp, {"mode": m}, out=hout, sparse=False)
            ms_m = (time.perf_counter() - t) / reps * 1e3
            paper[m] = {"e2e_ms": ms_m, "rays_per_s": nr / (ms_m * 1e-3), "paper_ms": pms, "paper_source": src,
                        "speedup_vs_paper": pms / ms_m}
        del hVp, hTp, hSp, hEp

    cpu, parity = None, None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu, ref = cpu_baseline(V, T, S, E, sample=args.cpu_sample)
        # parity on the sample the oracle just computed: the GPU outputs of all
        # three modes for the same rays of the timed workload (same kernels and
        # launch configuration as the timed steps)
        k = len(ref["hit"])
        # the outputs the LAST TIMED STEP of each mode wrote (overlapped steps,
        # full-size launch), sliced to the oracle's sample; a mode that was not
        # timed (--no-extra-modes) is recomputed on the same handle
        got = gpu_outputs(h, Sd[:k], Ed[:k])
        timed_src = []
        for m, fields in (("boolean", ("hit",)), ("intercept_count", ("count",)),
                          ("barycentric", ("tri", "t", "dist", "point"))):
            if m in last_out:
                got.update({f: last_out[m][f][:k].cpu().numpy() for f in fields})
                timed_src.append(m)
        parity = {"bench": parity_report(got, ref, S[:k], E[:k], f"{args.workload} N_t={len(T)}, "
                                                                   f"first {k} rays of the timed workload")}
        parity["bench"]["outputs"] = (f"last timed step's outputs of {', '.join(timed_src)}"
                                      if timed_src else "recomputed on the timed handle")
        if not args.no_parity:  # the 1e6-triangle mesh of configs[4] (L2-sized tree)
            V1, T1, S1, E1 = workload_inputs("sphere1m", 20_000, 0)
            ref1 = oracle_run(V1, T1, S1, E1)
            V1d, T1d = torch.from_numpy(V1).to(dev), torch.from_numpy(T1).to(dev)
            with rsi.rsi_build(V1d, T1d) as h1:
                got1 = gpu_outputs(h1, torch.from_numpy(S1).to(dev), torch.from_numpy(E1).to(dev))
            parity["sphere1m"] = parity_report(got1, ref1, S1, E1, f"sphere1m N_t={len(T1)}, 20000 rays")

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded UV-sphere mesh, uniform segments; see DESIGN.md 4)",
            "config": arm_config(args, len(T), world, backend),
            "build_ms": build_ms, "query_ms": query_ms, "serial": serial,
            "roofline": roofline(args.mode, n, query_ms, clk["sm_mhz"] if clk else None, work, args.workload),
            "work_per_ray": work,
            "cpu_baseline": cpu, "e2e": e2e, "parity": parity,
            "gpu_launches": launches,
            "gpu_launches_note": "rsi_launch_count() difference over the timed region (library kernels: "
                                 "BVH build chain + 1 traversal kernel per step)",
            "clocks": clk, "modes": extra, "configs_other": other, "paper_comparable": paper, "stats": stats,
        }
        print(json.dumps(line), flush=True)
    h.free()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
