"""Model of k-wide BVH collapses on the tree the GPU builds (GPU box; one-off
experiment quoted in DESIGN.md section 7).

For a sample of the bench segments, every binary node whose box the segment
enters and whose ancestors' boxes it all enters is "reached" (exact fp64 slab
test on the stored fp32 boxes).  A 2^L-wide walk visits the reached internal
nodes at depths 0, L, 2L, ... (a leaf child stands for itself), testing the
boxes of their up-to-2^L descendants L levels down.  Reported per segment
(all-hits traversal, i.e. intercept_count; independent of child order):
visits and child-box tests for L = 1 (binary), 2 (the 4-wide records), 3 (8-wide).
Usage: python tools/wide_model.py [workload] [n_rays]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_2305_01867_b200 import rsi

wl = sys.argv[1] if len(sys.argv) > 1 else "sphere"
nr = int(sys.argv[2]) if len(sys.argv) > 2 else 4000
V, T, S, E, _ = synth.workload(wl, nr, seed=3)
dev = torch.device("cuda:0")
h = rsi.rsi_build(torch.from_numpy(V).to(dev), torch.from_numpy(T).to(dev))
d = rsi.rsi_bvh_download(h)
child, box, root = d["child"], d["box"].astype(np.float64), d["root"]
nn = len(child)

# depth of every internal node, top-down
depth = np.full(nn, -1, np.int64)
depth[root] = 0
order = [root]
for n in order:
    for c in child[n]:
        if c >= 0:
            depth[c] = depth[n] + 1
            order.append(c)
order = np.array(order)



def enters(b, O, inv):  # b: [nn, 6] boxes; returns [nn, nr] segment-enters-box
    t0 = (b[:, None, 0:3] - O[None]) * inv[None]
    t1 = (b[:, None, 3:6] - O[None]) * inv[None]
    t0 = np.where(np.isnan(t0), -np.inf, t0)
    t1 = np.where(np.isnan(t1), np.inf, t1)
    tn = np.maximum(np.minimum(t0, t1).max(-1), 0.0)
    tf = np.minimum(np.maximum(t0, t1).min(-1), 1.0)
    return tn <= tf


reach_count = np.zeros(nn, np.int64)  # rays reaching each internal node
leaves_reached = 0
for c0 in range(0, nr, 256):
    O = S[c0:c0 + 256].astype(np.float64)
    D = E[c0:c0 + 256].astype(np.float64) - O
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = 1.0 / D
    hitc = [enters(box[:, s], O, inv) for s in (0, 1)]  # [nn, chunk] per child slot
    reached = np.zeros((nn, len(O)), bool)
    reached[root] = True
    for n in order:  # parents before children
        for s in (0, 1):
            c = child[n, s]
            if c >= 0:
                reached[c] = reached[n] & hitc[s][n]
    leaves_reached += sum(((child[:, s] < 0)[:, None] & reached & hitc[s]).sum() for s in (0, 1))
    reach_count += reached.sum(1)
leaves_reached /= nr


def n_desc(n, L):  # boxes a 2^L-wide record of node n holds
    if L == 0:
        return 1
    return sum(n_desc(c, L - 1) if c >= 0 else 1 for c in child[n])


parent = d["parent"]


def area(c):
    b = box[parent[c] >> 1, parent[c] & 1]
    e = np.maximum(b[3:6] - b[0:3], 0.0)
    return e[0] * e[1] + e[1] * e[2] + e[2] * e[0]


nleaf = np.zeros(nn, np.int64)
for n in order[::-1]:
    nleaf[n] = sum(nleaf[c] if c >= 0 else 1 for c in child[n])
KEYS = {"area": area, "leaves": lambda c: nleaf[c], "area*log2(leaves)": lambda c: area(c) * np.log2(nleaf[c] + 1)}
key = area


def greedy_cut(n, k):  # expand the internal member with the largest key until k members
    cut = [int(c) for c in child[n]]
    while len(cut) < k:
        inner = [c for c in cut if c >= 0]
        if not inner:
            break
        c = max(inner, key=key)
        cut.remove(c)
        cut += [int(x) for x in child[c]]
    return cut


def greedy(k):
    recs, widths, i = [root], [], 0
    while i < len(recs):
        cut = greedy_cut(recs[i], k)
        widths.append(len(cut))
        recs += [c for c in cut if c >= 0]
        i += 1
    recs, widths = np.array(recs), np.array(widths)
    vis = reach_count[recs]
    return vis.sum() / nr, (vis * widths).sum() / nr, widths.mean()


print(f"{wl}: N_t={len(T)}, nodes={nn}, max depth={depth.max()}, rays={nr}, leaves entered/ray={leaves_reached:.2f}")
for L in (1, 2, 3):
    sel = np.nonzero(depth % L == 0)[0]
    vis = reach_count[sel]
    w = np.array([n_desc(n, L) for n in sel])
    print(f"  {2 ** L}-wide: visits/ray {vis.sum() / nr:7.2f}   child-box tests/ray {(vis * w).sum() / nr:7.2f}   "
          f"mean children/record {w.mean():.2f}")
for k in (4, 8):
    for kname, kf in KEYS.items():
        key = kf
        v, t, m = greedy(k)
        print(f"  {k}-wide greedy cut by {kname}: visits/ray {v:7.2f}   child-box tests/ray {t:7.2f}   "
              f"mean children/record {m:.2f}")
