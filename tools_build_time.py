"""Time rsi_rebuild for the bench mesh (CUDA events, 20 iterations)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch, synth
from paper_2305_01867_b200 import rsi
for name in os.environ.get("WLS", "sphere").split(","):
    V, T, S, E, _ = synth.workload(name, 10, seed=3)
    Vd, Td = torch.from_numpy(V).cuda(), torch.from_numpy(T).cuda()
    h = rsi.rsi_build(Vd, Td)
    for _ in range(3): rsi.rsi_rebuild(h, Vd, Td)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    import time
    t = time.perf_counter(); e0.record()
    for _ in range(20): rsi.rsi_rebuild(h, Vd, Td)
    e1.record(); torch.cuda.synchronize()
    print(name, len(T), "rebuild ms (events):", e0.elapsed_time(e1) / 20, "wall ms:", (time.perf_counter() - t) / 20 * 1e3)
