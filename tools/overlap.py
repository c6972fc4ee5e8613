import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2305_01867_b200 import rsi
n = 10_000_000
V, T, S, E, _ = synth.workload("sphere", n, seed=3)
hS, hE = torch.from_numpy(S).pin_memory(), torch.from_numpy(E).pin_memory()
Vd, Td = torch.from_numpy(V).cuda(), torch.from_numpy(T).cuda()
dS, dE = torch.from_numpy(S).cuda(), torch.from_numpy(E).cuda()
bS, bE = torch.empty_like(dS), torch.empty_like(dE)
h = rsi.rsi_build(Vd, Td); o = rsi.alloc_outputs(n, "boolean", "cuda")
cs = torch.cuda.Stream(); ks = torch.cuda.Stream()
def tm(f, k=5):
    for _ in range(2): f()
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(k): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t) / k * 1e3
def copy_only():
    with torch.cuda.stream(cs): bS.copy_(hS, non_blocking=True); bE.copy_(hE, non_blocking=True)
def kern_only():
    with torch.cuda.stream(ks): rsi.rsi_intersect(h, dS, dE, "boolean", out=o)
def both():
    copy_only(); kern_only()
print("copy", tm(copy_only), "kernel", tm(kern_only), "both (2 streams)", tm(both))
# same with default stream kernel
def both0():
    copy_only(); rsi.rsi_intersect(h, dS, dE, "boolean", out=o)
print("both (copy side stream, kernel default stream)", tm(both0))
