"""GPU-box report (tests-style infrastructure: uses the oracle): for each
workload, the CUDA path vs the exhaustive fp64 oracle on every ray, with the
oracle's ambiguity flags COUNTED AND REPORTED per category (north_star: rays
within 1e-6 of an edge/vertex are counted, not hidden).  Mismatches are
counted over ALL rays, flagged or not.  Writes a text table to stdout."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
from paper_2305_01867_b200 import rsi

dev = torch.device("cuda:0")


def adversarial(V, T, n, seed):
    """Segments through mesh vertices and edge midpoints (edge/vertex flags)."""
    rng = np.random.default_rng(seed)
    tri = V[T[rng.integers(0, len(T), n)]]
    w = rng.integers(0, 2, (n, 1)).astype(np.float32)
    p = np.where(w > 0, tri[:, 0], 0.5 * (tri[:, 0] + tri[:, 1])).astype(np.float32)
    d = rng.normal(size=(n, 3)).astype(np.float32)
    return (p - d).astype(np.float32), (p + d).astype(np.float32)


cases = []
for name, nr in (("cube", 10_000), ("sphere", 200_000), ("terrain", 100_000), ("paper_terrain", 100_000)):
    V, T, S, E, _ = synth.workload(name, nr, seed=11)
    cases.append((f"{name} ({nr} rays)", V, T, S, E))
V, T = synth.uv_sphere()
S, E = adversarial(V, T, 20_000, 12)
cases.append(("sphere, rays through vertices / edge midpoints (20000)", V, T, S, E))
V, T = synth.fixture()
S, E = synth.fixture_rays()
cases.append(("Fig. 3 fixture (8 rays)", V, T, S, E))

names = [(oracle.FLAG_E, "E"), (oracle.FLAG_T, "T"), (oracle.FLAG_P, "P"), (oracle.FLAG_B, "B"), (oracle.FLAG_D, "D")]
print("# CUDA path vs exhaustive fp64 oracle, every ray; flags: E edge/vertex, T endpoint touch, P near-parallel,")
print("# B nearest tie, D dedup ambiguity (delta = 1e-6, DESIGN.md 2).  'mism' = rays whose boolean / count /")
print("# nearest-triangle differ (over ALL rays, flagged included); max|dt| over hit rays.")
print(f"{'workload':58s} {'rays':>7s} {'flagged':>8s} " + " ".join(f"{n:>6s}" for _, n in names)
      + f" {'mism_bool':>9s} {'mism_cnt':>8s} {'mism_tri':>8s} {'max|dt|':>9s}")
for label, V, T, S, E in cases:
    ref = oracle.run(V, T, S, E)
    Vd, Td, Sd, Ed = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (V, T, S, E))
    h = rsi.rsi_build(Vd, Td)
    hit = rsi.rsi_intersect(h, Sd, Ed, "boolean")["hit"].cpu().numpy()
    cnt = rsi.rsi_intersect(h, Sd, Ed, "intercept_count")["count"].cpu().numpy()
    bar = {k: v.cpu().numpy() for k, v in rsi.rsi_intersect(h, Sd, Ed, "barycentric").items()}
    h.free()
    fl = ref["flags"]
    m = ref["tri"] >= 0
    dt = float(np.abs(bar["t"][m] - ref["t"][m]).max()) if m.any() else 0.0
    print(f"{label:58s} {len(S):7d} {int((fl != 0).sum()):8d} "
          + " ".join(f"{int(((fl & b) != 0).sum()):6d}" for b, _ in names)
          + f" {int((hit != ref['hit']).sum()):9d} {int((cnt != ref['count']).sum()):8d}"
          + f" {int((bar['tri'] != ref['tri']).sum()):8d} {dt:9.2e}", flush=True)
