"""GPU-box probe: PCIe ceiling for barycentric's end-to-end step -- 300 MB
host->device and 300 MB device->host (1.25e7 segments x 24 B in, 24 B out),
alone and concurrently on two streams, pinned host memory, CUDA events."""
import json, torch

n = 300_000_000
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
cur = torch.cuda.current_stream()


def timed(kind):
    best = 1e9
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cur)
        for s in (s1, s2):
            s.wait_stream(cur)
        if kind in ("h2d", "both"):
            with torch.cuda.stream(s1):
                d_in.copy_(h_in, non_blocking=True)
        if kind in ("d2h", "both"):
            with torch.cuda.stream(s2):
                h_out.copy_(d_out, non_blocking=True)
        for s in (s1, s2):
            cur.wait_stream(s)
        b.record(cur)
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


r = {k: round(timed(k), 3) for k in ("h2d", "d2h", "both")}
r["GBps"] = {k: round(n / (v * 1e-3) / 1e9, 1) for k, v in r.items() if k != "GBps"}
print(json.dumps(r))
