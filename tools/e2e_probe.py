"""GPU-box probe: end-to-end rsi_test time (pinned host buffers, dense outputs)
per mode, as bench.py's e2e leg; run under RSI_TEST_* env variants."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2305_01867_b200 import rsi

n = int(os.environ.get("N", "12500000"))
V, T, S, E, _ = synth.workload(os.environ.get("WL", "sphere"), n, seed=3)
pin = lambda a: torch.from_numpy(a).pin_memory()  # noqa: E731
hV, hT, hS, hE = pin(V), pin(T), pin(S), pin(E)
res = {"env": {k: v for k, v in os.environ.items() if k.startswith("RSI_TEST")}}
for mode in os.environ.get("MODES", "boolean,barycentric").split(","):
    hout = {k: v.pin_memory() for k, v in rsi.alloc_outputs(n, mode, "cpu").items()}
    for _ in range(2):
        rsi.rsi_test(hV, hT, hS, hE, {"mode": mode}, out=hout, sparse=False)
    best = []
    for _ in range(3):
        t = time.perf_counter()
        for _ in range(5):
            rsi.rsi_test(hV, hT, hS, hE, {"mode": mode}, out=hout, sparse=False)
        best.append((time.perf_counter() - t) / 5 * 1e3)
    res[mode] = {"ms": round(min(best), 3), "Grays_s": round(n / min(best) / 1e6, 3)}
print(json.dumps(res))
