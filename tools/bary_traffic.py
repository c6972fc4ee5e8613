"""GPU-box diagnostic (run under ncu --metrics dram__bytes_*): barycentric
launches with different output subsets, to attribute DRAM write traffic."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2305_01867_b200 import rsi

n = int(os.environ.get("N", "10000000"))
V, T, S, E, _ = synth.workload("sphere", n, seed=3)
dev = torch.device("cuda:0")
Vd, Td, Sd, Ed = (torch.from_numpy(a).to(dev) for a in (V, T, S, E))
h = rsi.rsi_build(Vd, Td)
full = rsi.alloc_outputs(n, "barycentric", dev)
for label, keys in (("tri", ("tri",)), ("tri_t", ("tri", "t")), ("tri_t_dist", ("tri", "t", "dist")), ("full", ("tri", "t", "dist", "point"))):
    out = {k: full[k] for k in keys}
    for _ in range(2):
        rsi.rsi_intersect(h, Sd, Ed, "barycentric", out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rsi.rsi_intersect(h, Sd, Ed, "barycentric", out=out)
    e1.record(); torch.cuda.synchronize()
    print(label, f"{e0.elapsed_time(e1):.3f} ms", flush=True)
