import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2305_01867_b200 import rsi
n = 10_000_000
V, T, S, E, _ = synth.workload("sphere", n, seed=3)
pin = lambda a: torch.from_numpy(a).pin_memory()
hV, hT, hS, hE = pin(V), pin(T), pin(S), pin(E)
out = {"hit": torch.empty(n, dtype=torch.uint8).pin_memory()}
for ch in [262144, 1 << 20, 1 << 21, 1 << 22, n]:
    os.environ["RSI_TEST_CHUNK"] = str(ch)
    for _ in range(2): rsi.rsi_test(hV, hT, hS, hE, {"mode": "boolean"}, out=out)
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(5): rsi.rsi_test(hV, hT, hS, hE, {"mode": "boolean"}, out=out)
    torch.cuda.synchronize(); print("chunk", ch, "ms", (time.perf_counter() - t) / 5 * 1e3)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(2): rsi.rsi_test(hV, hT, hS, hE, {"mode": "boolean"}, out=out, stream=s)
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(5): rsi.rsi_test(hV, hT, hS, hE, {"mode": "boolean"}, out=out, stream=s)
    torch.cuda.synchronize(); print("non-default stream, last chunk", "ms", (time.perf_counter() - t) / 5 * 1e3)
