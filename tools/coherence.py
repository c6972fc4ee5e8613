"""GPU-box experiment: traversal time on randomly ordered vs spatially sorted
segments (6-D Morton order of (start, end)), to bound what ray reordering buys."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2305_01867_b200 import rsi

n = int(os.environ.get("N", "10000000"))
wl = os.environ.get("WL", "sphere")
V, T, S, E, _ = synth.workload(wl, n, seed=3)

def key6(S, E, bits):
    P = np.concatenate([S, E], 1).astype(np.float64)
    lo, hi = P.min(0), P.max(0)
    q = np.clip(((P - lo) / np.maximum(hi - lo, 1e-30) * (1 << bits)).astype(np.int64), 0, (1 << bits) - 1)
    k = np.zeros(len(S), np.int64)
    for b in range(bits - 1, -1, -1):
        for a in range(6):
            k = (k << 1) | ((q[:, a] >> b) & 1)
    return k

dev = torch.device("cuda:0")
Vd, Td = torch.from_numpy(V).to(dev), torch.from_numpy(T).to(dev)
h = rsi.rsi_build(Vd, Td)
for label, bits in (("random", 0), ("morton6x3", 3), ("morton6x5", 5), ("morton6x8", 8)):
    if bits:
        o = np.argsort(key6(S, E, bits), kind="stable")
        S2, E2 = np.ascontiguousarray(S[o]), np.ascontiguousarray(E[o])
    else:
        S2, E2 = S, E
    Sd, Ed = torch.from_numpy(S2).to(dev), torch.from_numpy(E2).to(dev)
    for mode in ("boolean", "barycentric", "intercept_count"):
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
        print(f"{wl} {label} {mode} {ms:.3f} ms {n/ms/1e6:.3f} Grays/s", flush=True)
