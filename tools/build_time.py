"""GPU-box helper: device time of rsi_rebuild (deferred status, CUDA events,
20 iterations) for named workloads and random meshes, default vs Apetrei build."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_2305_01867_b200 import rsi

def meshes():
    for name in os.environ.get("WLS", "sphere,paper_terrain,sphere1m").split(","):
        V, T, *_ = synth.workload(name, 10, seed=3)
        yield name, V, T
    for nt in (int(x) for x in os.environ.get("NTS", "20000,40000,65536,200000").split(",") if x):
        rng = np.random.default_rng(nt)
        V = rng.uniform(-1, 1, (3 * nt, 3)).astype(np.float32)
        yield f"random{nt}", V, np.arange(3 * nt, dtype=np.int32).reshape(nt, 3)

for name, V, T in meshes():
    Vd, Td = torch.from_numpy(V).cuda(), torch.from_numpy(T).cuda()
    for ap in (False, True):
        h = rsi.rsi_build(Vd, Td, rsi.Options(apetrei=ap, deferred_status=True))
        for _ in range(3):
            rsi.rsi_rebuild(h, Vd, Td)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            rsi.rsi_rebuild(h, Vd, Td)
        e1.record()
        torch.cuda.synchronize()
        assert rsi.rsi_validate(h)["ok"]
        print(f"{name} N_t={len(T)} {'apetrei' if ap else 'karras'} rebuild {e0.elapsed_time(e1) / 20:.3f} ms", flush=True)
        h.free()
