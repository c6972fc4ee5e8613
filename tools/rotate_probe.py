"""GPU-box probe: RSI_OPT_ROTATE vs default -- rebuild time, query time per
mode, box tests per ray, validator, parity on a sample."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_2305_01867_b200 import rsi

dev = torch.device("cuda:0")
for wl in ("sphere", "paper_terrain", "terrain", "sphere1m"):
    n = 10_000_000
    V, T, S, E, _ = synth.workload(wl, n, seed=3)
    Vd, Td, Sd, Ed = (torch.from_numpy(a).to(dev) for a in (V, T, S, E))
    res = {}
    for rot in (False, True):
        h = rsi.rsi_build(Vd, Td, rsi.Options(rotate=rot, deferred_status=True))
        for _ in range(3):
            rsi.rsi_rebuild(h, Vd, Td)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            rsi.rsi_rebuild(h, Vd, Td)
        e1.record(); torch.cuda.synchronize()
        line = {"rebuild_ms": round(e0.elapsed_time(e1) / 10, 4)}
        assert rsi.rsi_validate(h)["ok"]
        for mode in ("boolean", "barycentric", "intercept_count"):
            out = rsi.alloc_outputs(n, mode, dev)
            for _ in range(2):
                rsi.rsi_intersect(h, Sd, Ed, mode, out=out)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(5):
                rsi.rsi_intersect(h, Sd, Ed, mode, out=out)
            e1.record(); torch.cuda.synchronize()
            line[mode] = round(e0.elapsed_time(e1) / 5, 4)
            res.setdefault(mode, []).append(out)
        h.free()
        hc = rsi.rsi_build(Vd, Td, rsi.Options(rotate=rot, counters=True))
        rsi.rsi_intersect(hc, Sd, Ed, "boolean")
        st = rsi.rsi_get_stats(hc)
        line["box_per_ray"] = round(st["box_tests"] / n, 3)
        hc.free()
        print(wl, "rotate" if rot else "default", line, flush=True)
    for mode, (a, b) in res.items():
        for k in a:
            x, y = a[k], b[k]
            same = torch.equal(x, y) if x.dtype != torch.float32 else bool(((x == y) | (torch.isnan(x) & torch.isnan(y))).all())
            assert same or k in ("t", "dist", "point"), (wl, mode, k)
