"""GPU-box report (test infrastructure: uses the oracle): EVERY segment of the
bench workload (sphere N_t = 1e4, 1.25e7 segments, bench.py's seed) and of
configs[3] (folded terrain, 1e7 segments) -- GPU outputs of one full-size
launch per mode against the exhaustive fp64 oracle, compared in chunks of
1e6 segments (bench.parity_report per chunk, summed).  Prints one JSON line
per workload."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
import bench
from paper_2305_01867_b200 import rsi

dev = torch.device("cuda:0")
# WLS="name:n,name:n" selects other workloads (e.g. paper_terrain:10000000,sphere1m:200000)
WLS = [(w.split(":")[0], int(w.split(":")[1])) for w in
       os.environ.get("WLS", "sphere:12500000,terrain:10000000").split(",")]
for name, n in WLS:
    V, T, S, E = bench.workload_inputs(name, n, 0)
    Vd, Td, Sd, Ed = (torch.from_numpy(a).to(dev) for a in (V, T, S, E))
    h = rsi.rsi_build(Vd, Td)
    got = {"hit": rsi.rsi_intersect(h, Sd, Ed, "boolean")["hit"].cpu().numpy(),
           "count": rsi.rsi_intersect(h, Sd, Ed, "intercept_count")["count"].cpu().numpy()}
    got.update({k: v.cpu().numpy() for k, v in rsi.rsi_intersect(h, Sd, Ed, "barycentric").items()})
    h.free()
    tot = None
    t0 = time.perf_counter()
    step = 1_000_000 if len(T) < 100_000 else 20_000
    for a in range(0, n, step):
        b = min(n, a + step)
        ref = oracle.run(V, T, S[a:b], E[a:b])
        r = bench.parity_report({k: v[a:b] for k, v in got.items()}, ref, S[a:b], E[a:b], name)
        if tot is None:
            tot = r
        else:
            for k in ("rays", "mismatch_bool", "mismatch_count", "mismatch_tri", "tol_violations", "flagged_mismatch"):
                tot[k] += r[k]
            for k in ("max_dt", "max_ddist_rel", "max_dpoint_rel"):
                tot[k] = max(tot[k], r[k])
            for k in tot["flagged"]:
                tot["flagged"][k] += r["flagged"][k]
            tot["ok"] = tot["ok"] and r["ok"]
    tot["workload"] = f"{name} N_t={len(T)}, all {n} segments (bench.py seed), one launch per mode"
    tot["oracle_s"] = round(time.perf_counter() - t0, 1)
    tot["oracle_cores"] = oracle.max_threads()
    print(json.dumps(tot), flush=True)
