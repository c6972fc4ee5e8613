import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2305_01867_b200 import rsi
n = 10_000_000
V, T, S, E, _ = synth.workload("sphere", n, seed=3)
pin = lambda a: torch.from_numpy(a).pin_memory()
hV, hT, hS, hE = pin(V), pin(T), pin(S), pin(E)
out = {"hit": torch.empty(n, dtype=torch.uint8).pin_memory()}
for _ in range(3): rsi.rsi_test(hV, hT, hS, hE, {"mode": "boolean"}, out=out)
os.environ["RSI_TEST_TRACE"] = "1"
for _ in range(3):
    t = time.perf_counter(); rsi.rsi_test(hV, hT, hS, hE, {"mode": "boolean"}, out=out); print("call ms", (time.perf_counter() - t) * 1e3, flush=True)
