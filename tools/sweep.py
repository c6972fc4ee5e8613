"""GPU-box helper: time the traversal per mode for several knob settings."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2305_01867_b200 import rsi

n = int(os.environ.get("N", "10000000"))
wl = os.environ.get("WL", "sphere")
V, T, S, E, _ = synth.workload(wl, n, seed=3)
dev = torch.device("cuda:0")
Vd, Td, Sd, Ed = (torch.from_numpy(a).to(dev) for a in (V, T, S, E))
res = {}
MODES = os.environ.get("MODES", "boolean,barycentric,intercept_count").split(",")
for cfg in os.environ.get("CFGS", "-1:1").split(","):
    mt, sp = cfg.split(":")
    os.environ["RSI_MIN_TRAV"] = mt
    os.environ["RSI_SPEC"] = sp
    h = rsi.rsi_build(Vd, Td)
    for mode in MODES:
        out = rsi.alloc_outputs(n, mode, dev)
        for _ in range(2):
            rsi.rsi_intersect(h, Sd, Ed, mode, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            rsi.rsi_intersect(h, Sd, Ed, mode, out=out)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        res[f"{os.path.basename(os.environ.get('RSI_LIB', 'default'))}:{mode}/min_trav={mt},spec={sp}"] = {"ms": round(ms, 3), "Grays_s": round(n / ms / 1e6, 3)}
    h.free()
if os.environ.get("COUNTERS", "1") == "0":
    [print(k, json.dumps(v)) for k, v in res.items()]; sys.exit(0)
hc = rsi.rsi_build(Vd, Td, rsi.Options(counters=True))
for mode in MODES:
    rsi.rsi_reset_stats(hc)
    rsi.rsi_intersect(hc, Sd, Ed, mode)
    st = rsi.rsi_get_stats(hc)
    res[f"work/{mode}"] = {"box_per_ray": st["box_tests"] / n, "mt_per_ray": st["mt_tests"] / n,
                           "fp64_pairs": st["fp64_pairs"], "fp64_rays": st["fp64_rays"], "overflow": st["overflow_rays"],
                           "trav_eff": st["it_search"] / max(1, 32 * st["iterations"]),
                           "trav_pend": st["it_pending"] / max(1, 32 * st["iterations"]),
                           "trav_idle": st["it_idle"] / max(1, 32 * st["iterations"]),
                           "iters_per_ray": st["iterations"] * 32 / n,
                           "leaf_eff": st["leaf_lanes"] / max(1, 32 * st["leaf_phases"])}
[print(k, json.dumps(v)) for k, v in res.items()]
