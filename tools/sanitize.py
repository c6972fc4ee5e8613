"""Small end-to-end run of every kernel for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_2305_01867_b200 import rsi
dev = "cuda:0"
for name, nt_rays in (("fixture", None), ("cube", 3000), ("sphere", 5000)):
    if name == "fixture":
        V, T = synth.canopy(); S, E = synth.fixture_rays()
    else:
        V, T, S, E, _ = synth.workload(name, nt_rays, seed=1)
    Vd, Td, Sd, Ed = (torch.from_numpy(a).to(dev) for a in (V, T, S, E))
    h = rsi.rsi_build(Vd, Td)
    for m in ("boolean", "barycentric", "intercept_count"):
        o = rsi.rsi_intersect(h, Sd, Ed, m)
    rsi.sparse_barycentric(rsi.rsi_intersect(h, Sd, Ed, "barycentric"))
    rsi.rsi_bvh_download(h)
    h.free()
# overflow re-pass + multi-block sort path
V = np.vstack([np.float32([[0, 0, 0.1 * k], [1, 0, 0.1 * k], [0, 1, 0.1 * k]]) for k in range(12)]).astype(np.float32)
T = np.arange(36, dtype=np.int32).reshape(12, 3)
S = np.float32([[0.2, 0.2, -1.0]] * 40); E = np.float32([[0.2, 0.2, 5.0]] * 40)
h = rsi.rsi_build(torch.from_numpy(V).to(dev), torch.from_numpy(T).to(dev))
c = rsi.rsi_intersect(h, torch.from_numpy(S).to(dev), torch.from_numpy(E).to(dev), "intercept_count")["count"].cpu()
assert (c == 12).all(), c
h.free()
rng = np.random.default_rng(1)
V = rng.uniform(0, 1, (3 * 70001, 3)).astype(np.float32); T = np.arange(3 * 70001, dtype=np.int32).reshape(-1, 3)
h = rsi.rsi_build(torch.from_numpy(V).to(dev), torch.from_numpy(T).to(dev)); h.free()
# RSI_OPT_APETREI (63-bit codes, two sorts, agglomerative build) on the rank-sort
# and multi-block sizes, queried in every mode; validator; fault injection
for nt in (5000, 70001):
    Vd = torch.from_numpy(V[:3 * nt]).to(dev); Td = torch.from_numpy(T[:nt]).to(dev)
    h = rsi.rsi_build(Vd, Td, rsi.Options(apetrei=True))
    Sd, Ed = (torch.from_numpy(a).to(dev) for a in synth.box_rays(3000, -0.2, 1.2, seed=3))
    for m in ("boolean", "barycentric", "intercept_count"):
        rsi.rsi_intersect(h, Sd, Ed, m)
    assert rsi.rsi_validate(h)["ok"]
    rsi.rsi_bvh_download(h)
    h.free()
for nt in (5000, 70001):  # refit with rotations; sparse end-to-end path
    Vd = torch.from_numpy(V[:3 * nt]).to(dev); Td = torch.from_numpy(T[:nt]).to(dev)
    h = rsi.rsi_build(Vd, Td, rsi.Options(rotate=True))
    assert rsi.rsi_validate(h)["ok"]
    rsi.rsi_intersect(h, Sd, Ed, "barycentric")
    h.free()
rsi.rsi_test(V[:15000], T[:5000], *synth.box_rays(3000, -0.2, 1.2, seed=4), {"mode": "barycentric"})
h = rsi.rsi_build(Vd, Td, rsi.Options(apetrei=True, debug_refit_leaves=20000))
assert not rsi.rsi_validate(h)["ok"]
rsi.rsi_intersect(h, Sd, Ed, "boolean")
h.free()
hv = rsi.rsi_test(*synth.workload("sphere", 3000, seed=2)[:4], {"mode": "boolean"})
rsi.rsi_release_cache()
torch.cuda.synchronize()
print("sanitize run ok")
# round 2: SAH subtrees (N_t <= 32768, every mode), the treelet refit path
# (32769 .. 65536), and rsi_bvh_upload (round trip of the downloaded tree)
for nt in (20000, 40000):
    Vd = torch.from_numpy(V[:3 * nt]).to(dev); Td = torch.from_numpy(T[:nt]).to(dev)
    h = rsi.rsi_build(Vd, Td)
    Sd, Ed = (torch.from_numpy(a).to(dev) for a in synth.box_rays(3000, -0.2, 1.2, seed=4))
    for m in ("boolean", "barycentric", "intercept_count"):
        rsi.rsi_intersect(h, Sd, Ed, m)
    d = rsi.rsi_bvh_download(h)
    rsi.rsi_bvh_upload(h, d["child"], d["box"], d["leaf_tri"], 0)
    rsi.rsi_intersect(h, Sd, Ed, "barycentric")
    assert rsi.rsi_validate(h)["ok"]
    h.free()
print("sanitize round-2 paths ok")
# bench.py's overlapped steps: two handles on two streams, rebuild + intersect
# alternating with no host sync (step k+1's build runs beside step k's walk)
V2, T2, S2, E2, _ = synth.workload("sphere", 20000, seed=5)
Vd, Td, Sd, Ed = (torch.from_numpy(a).to(dev) for a in (V2, T2, S2, E2))
hs = [rsi.rsi_build(Vd, Td, rsi.Options(deferred_status=True)) for _ in range(2)]
sts = [torch.cuda.Stream(), torch.cuda.Stream()]
for k in range(4):
    with torch.cuda.stream(sts[k % 2]):
        rsi.rsi_rebuild(hs[k % 2], Vd, Td)
        for m in ("boolean", "barycentric", "intercept_count"):
            rsi.rsi_intersect(hs[k % 2], Sd, Ed, m)
torch.cuda.synchronize()
for h in hs:
    rsi.rsi_build_status(h)
    h.free()
print("sanitize overlapped steps ok")
