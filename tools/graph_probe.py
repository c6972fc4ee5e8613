"""GPU-box probe: device time of rsi_rebuild (deferred status) and of
rebuild + intersect, eager vs replayed from a captured CUDA graph."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2305_01867_b200 import rsi

dev = torch.device("cuda:0")
for name, nr in (("sphere", 1_000_000), ("sphere", 10_000_000)):
    V, T, S, E, _ = synth.workload(name, nr, seed=3)
    Vd, Td, Sd, Ed = (torch.from_numpy(a).to(dev) for a in (V, T, S, E))
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        h = rsi.rsi_build(Vd, Td, rsi.Options(deferred_status=True))
        out = rsi.alloc_outputs(nr, "boolean", dev)
        def step():
            rsi.rsi_rebuild(h, Vd, Td)
            rsi.rsi_intersect(h, Sd, Ed, "boolean", out=out)
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            step()
        for label, fn in (("eager", step), ("graph", g.replay)):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(20):
                fn()
            e1.record(s)
            torch.cuda.synchronize()
            print(f"{name} N_r={nr} {label}: {e0.elapsed_time(e1) / 20:.4f} ms/step", flush=True)
        hit_g = out["hit"].clone()
        step(); torch.cuda.synchronize()
        assert torch.equal(hit_g, out["hit"])
        rsi.rsi_build_status(h)
        h.free()
