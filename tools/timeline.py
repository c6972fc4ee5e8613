"""GPU-box helper: kernel timeline of bench steps (rsi_rebuild + rsi_intersect)
via torch.profiler (CUPTI): start offsets, durations and the gaps between."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
import synth
from paper_2305_01867_b200 import rsi

n = int(os.environ.get("N", "10000000"))
wl = os.environ.get("WL", "sphere")
mode = os.environ.get("MODE", "boolean")
V, T, S, E, _ = synth.workload(wl, n, seed=3)
dev = torch.device("cuda:0")
Vd, Td, Sd, Ed = (torch.from_numpy(a).to(dev) for a in (V, T, S, E))
h = rsi.rsi_build(Vd, Td)
out = rsi.alloc_outputs(n, mode, dev)
for _ in range(3):
    rsi.rsi_rebuild(h, Vd, Td); rsi.rsi_intersect(h, Sd, Ed, mode, out=out)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(3):
        rsi.rsi_rebuild(h, Vd, Td); rsi.rsi_intersect(h, Sd, Ed, mode, out=out)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0 = None
prev_end = None
for e in evs:
    st, en = e.time_range.start, e.time_range.end
    if t0 is None: t0 = st
    gap = (st - prev_end) if prev_end is not None else 0
    print(f"{(st - t0):10.1f} us  dur {en - st:9.1f}  gap {gap:7.1f}  {e.name[:60]}")
    prev_end = en
