"""GPU-box probe: visible rebuild time per overlapped step (two handles, two
streams, as bench.py) against the serial step, for build options that change
the rebuild chain's length.  Prints per option: serial build / query ms and
the overlapped step ms (visible rebuild = overlapped step - query)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2305_01867_b200 import rsi

n = int(os.environ.get("N", "12500000"))
wl = os.environ.get("WL", "sphere")
V, T, S, E, _ = synth.workload(wl, n, seed=3)
dev = torch.device("cuda:0")
Vd, Td, Sd, Ed = (torch.from_numpy(a).to(dev) for a in (V, T, S, E))
cur = torch.cuda.current_stream()
K = 10
for name, kw in (("default", {}), ("plain_tree", {"plain_tree": True})):
    hs = [rsi.rsi_build(Vd, Td, rsi.Options(deferred_status=True, **kw)) for _ in range(2)]
    outs = [rsi.alloc_outputs(n, "boolean", dev) for _ in range(2)]
    sts = [torch.cuda.Stream(), torch.cuda.Stream()]
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    # serial: per-step events
    bq = []
    for k in range(3 + K):
        a, b, c = ev(), ev(), ev()
        a.record(cur); rsi.rsi_rebuild(hs[0], Vd, Td); b.record(cur)
        rsi.rsi_intersect(hs[0], Sd, Ed, "boolean", out=outs[0]); c.record(cur)
        bq.append((a, b, c))
    torch.cuda.synchronize()
    bms = sum(a.elapsed_time(b) for a, b, c in bq[3:]) / K
    qms = sum(b.elapsed_time(c) for a, b, c in bq[3:]) / K
    def run(k):
        with torch.cuda.stream(sts[k % 2]):
            rsi.rsi_rebuild(hs[k % 2], Vd, Td)
            rsi.rsi_intersect(hs[k % 2], Sd, Ed, "boolean", out=outs[k % 2])
    for k in range(3):
        run(k)
    torch.cuda.synchronize()
    t0, t1 = ev(), ev()
    t0.record(cur)
    for st in sts:
        st.wait_stream(cur)
    for k in range(K):
        run(k)
    for st in sts:
        cur.wait_stream(st)
    t1.record(cur)
    torch.cuda.synchronize()
    oms = t0.elapsed_time(t1) / K
    print(json.dumps({"opt": name, "n": n, "build_ms": round(bms, 4), "query_ms": round(qms, 4),
                      "serial_step_ms": round(bms + qms, 4), "overlap_step_ms": round(oms, 4),
                      "visible_build_ms": round(oms - qms, 4)}))
    for h in hs:
        rsi.rsi_build_status(h)
        h.free()
