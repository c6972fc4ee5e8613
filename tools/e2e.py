import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2305_01867_b200 import rsi
n = 10_000_000
V, T, S, E, _ = synth.workload("sphere", n, seed=3)
pin = lambda a: torch.from_numpy(a).pin_memory()
hV, hT, hS, hE = pin(V), pin(T), pin(S), pin(E)
out = {"hit": torch.empty(n, dtype=torch.uint8).pin_memory()}
def tm(f, k=5):
    for _ in range(2): f()
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(k): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t) / k * 1e3
print("rsi_test full      ms", tm(lambda: rsi.rsi_test(hV, hT, hS, hE, {"mode": "boolean"}, out=out)))
small = {"hit": torch.empty(1000, dtype=torch.uint8).pin_memory()}
print("rsi_test 1e3 rays  ms", tm(lambda: rsi.rsi_test(hV, hT, hS[:1000], hE[:1000], {"mode": "boolean"}, out=small)))
dS, dE = torch.empty(n, 3, device="cuda"), torch.empty(n, 3, device="cuda")
def cp():
    dS.copy_(hS, non_blocking=True); dE.copy_(hE, non_blocking=True)
print("torch H2D S+E      ms", tm(cp))
Vd, Td = torch.from_numpy(V).cuda(), torch.from_numpy(T).cuda()
h = rsi.rsi_build(Vd, Td)
o = rsi.alloc_outputs(n, "boolean", "cuda")
print("intersect (dev)    ms", tm(lambda: rsi.rsi_intersect(h, dS, dE, "boolean", out=o)))
def manual():
    cp(); rsi.rsi_rebuild(h, Vd, Td); rsi.rsi_intersect(h, dS, dE, "boolean", out=o); out["hit"].copy_(o["hit"], non_blocking=True)
print("serial H2D+build+intersect+D2H ms", tm(manual))
os.environ["RSI_TEST_TRACE"] = "1"
rsi.rsi_test(hV, hT, hS, hE, {"mode": "boolean"}, out=out)
import ctypes
cudart = ctypes.CDLL("libcudart.so.12") if False else None
t = time.perf_counter(); rsi.rsi_test(hV, hT, hS, hE, {"mode": "boolean"}, out=out); print("traced call ms", (time.perf_counter()-t)*1e3)
