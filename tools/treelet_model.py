"""CPU model of BVH quality for the bench segments (no GPU; one-off experiment
quoted in DESIGN.md section 7).  Builds the LBVH the GPU builds (30-bit
z-major Morton codes with the reading-R8 extent floor, highest-differing-bit
splits = the Karras topology), optionally a binned-SAH tree and Karras &
Aila's treelet restructuring (exact DP over member subsets, largest-area
treelet formation, SAH constants Ci = 1.2, Ct = 1), collapses each into the
4-wide greedy-cut records the traversal walks, and counts per segment the
record visits and child-box tests of an all-hits walk (exact fp64 slab test).

Usage: python tools/treelet_model.py [workload] [treelet size] [passes]
"""
import sys, time
import numpy as np
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import synth
wl = sys.argv[1] if len(sys.argv) > 1 else "sphere"
nr = 3000
V, T, S, E, _ = synth.workload(wl, nr, seed=3)
tri = V[T].astype(np.float64)               # [N,3,3]
tlo, thi = tri.min(1), tri.max(1)
cen = tri.mean(1)
N = len(T)

def expand10(v):
    v = v.astype(np.uint64) & 0x3ff
    v = (v | (v << 16)) & 0x30000ff
    v = (v | (v << 8)) & 0x300f00f
    v = (v | (v << 4)) & 0x30c30c3
    v = (v | (v << 2)) & 0x9249249
    return v

def lbvh():
    lo, hi = tlo.min(0), thi.max(0)
    W = (hi - lo).max()
    w = np.maximum(hi - lo, W / 64)
    q = np.clip(np.floor((cen - lo) / w * 1024), 0, 1023).astype(np.uint64)
    code = expand10(q[:, 2]) | (expand10(q[:, 1]) << 1) | (expand10(q[:, 0]) << 2)
    order = np.argsort(code, kind="stable")
    codes = code[order]
    nodes = []  # (left, right) refs: >=0 internal, <0 ~leafidx(prim)
    def build(i, j):
        if i == j:
            return ~int(order[i])
        if codes[i] == codes[j]:
            m = (i + j) // 2
        else:
            x = int(codes[i]) ^ int(codes[j]); b = x.bit_length() - 1
            # last index with bit b equal to codes[i]'s
            lo_, hi_ = i, j
            while hi_ - lo_ > 1:
                mid = (lo_ + hi_) // 2
                if (int(codes[mid]) >> b) == (int(codes[i]) >> b): lo_ = mid
                else: hi_ = mid
            m = lo_
        k = len(nodes); nodes.append(None)
        nodes[k] = (build(i, m), build(m + 1, j))
        return k
    sys.setrecursionlimit(100000)
    r = build(0, N - 1)
    return nodes, r

def sah(nbins=32, maxleaf=1):
    nodes = []
    def area(lo, hi):
        e = np.maximum(hi - lo, 0); return e[..., 0]*e[..., 1] + e[..., 1]*e[..., 2] + e[..., 2]*e[..., 0]
    def build(idx):
        if len(idx) == 1:
            return ~int(idx[0])
        c = cen[idx]; clo, chi = c.min(0), c.max(0)
        best = (np.inf, None)
        for ax in range(3):
            if chi[ax] - clo[ax] <= 0: continue
            b = np.minimum(((c[:, ax] - clo[ax]) / (chi[ax] - clo[ax]) * nbins).astype(int), nbins - 1)
            blo = np.full((nbins, 3), np.inf); bhi = np.full((nbins, 3), -np.inf); cnt = np.zeros(nbins)
            for k in range(nbins):
                m = b == k
                if m.any():
                    blo[k] = tlo[idx[m]].min(0); bhi[k] = thi[idx[m]].max(0); cnt[k] = m.sum()
            plo = np.minimum.accumulate(blo); phi = np.maximum.accumulate(bhi); pc = np.cumsum(cnt)
            slo = np.minimum.accumulate(blo[::-1])[::-1]; shi = np.maximum.accumulate(bhi[::-1])[::-1]; sc = np.cumsum(cnt[::-1])[::-1]
            for k in range(nbins - 1):
                if pc[k] == 0 or sc[k + 1] == 0: continue
                cost = area(plo[k], phi[k]) * pc[k] + area(slo[k + 1], shi[k + 1]) * sc[k + 1]
                if cost < best[0]: best = (cost, (ax, b, k))
        if best[1] is None:
            m = len(idx) // 2; L, R = idx[:m], idx[m:]
        else:
            ax, b, k = best[1]; L, R = idx[b <= k], idx[b > k]
        kk = len(nodes); nodes.append(None)
        nodes[kk] = (build(L), build(R))
        return kk
    sys.setrecursionlimit(100000)
    r = build(np.arange(N))
    return nodes, r

def evaluate(nodes, root, label):
    nn = len(nodes)
    child = np.array(nodes, dtype=np.int64)
    # boxes of internal nodes
    blo = np.zeros((nn, 3)); bhi = np.zeros((nn, 3))
    order = [root]
    for n in order:
        for c in child[n]:
            if c >= 0: order.append(c)
    def cbox(c):
        return (tlo[~c], thi[~c]) if c < 0 else (blo[c], bhi[c])
    for n in order[::-1]:
        l, r = cbox(child[n, 0]), cbox(child[n, 1])
        blo[n] = np.minimum(l[0], r[0]); bhi[n] = np.maximum(l[1], r[1])
    # reach counts (exact slab)
    O = S.astype(np.float64); D = E.astype(np.float64) - O
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = 1.0 / D
    def enters(lo, hi):
        t0 = (lo[:, None] - O[None]) * inv[None]; t1 = (hi[:, None] - O[None]) * inv[None]
        t0 = np.where(np.isnan(t0), -np.inf, t0); t1 = np.where(np.isnan(t1), np.inf, t1)
        return np.maximum(np.minimum(t0, t1).max(-1), 0) <= np.minimum(np.maximum(t0, t1).min(-1), 1)
    ent = enters(blo, bhi)  # [nn, nr]
    leaf_ent = enters(tlo, thi)  # [N, nr]
    reach = np.zeros((nn, nr), bool); reach[root] = ent[root]
    for n in order:
        for c in child[n]:
            if c >= 0: reach[c] = reach[n] & ent[c]
    rc = reach.sum(1)
    # greedy 4-cut by area from each record node; a record visit happens if the record's node is reached
    def area_(c):
        lo, hi = cbox(c); e = np.maximum(hi - lo, 0); return e[0]*e[1]+e[1]*e[2]+e[2]*e[0]
    recs = [root]; vis = 0; tests = 0; i = 0
    while i < len(recs):
        n = recs[i]; i += 1
        cut = [int(c) for c in child[n]]
        while len(cut) < 4:
            inner = [c for c in cut if c >= 0]
            if not inner: break
            c = max(inner, key=area_); cut.remove(c); cut += [int(x) for x in child[c]]
        # a record is visited by rays reaching its node -- the root record by rays entering root box
        v = rc[n]; vis += v; tests += v * len(cut)
        recs += [c for c in cut if c >= 0]
    # leaves tested: leaf reached = parent reached & leaf box entered
    leaves = 0
    for n in order:
        for c in child[n]:
            if c < 0: leaves += (reach[n] & leaf_ent[~c]).sum()
    sa = sum(area_(n) for n in range(nn)) / area_(root)
    print(f"{label:8s} 4-wide visits/ray {vis/nr:6.2f}  box tests/ray {tests/nr:6.2f}  leaves/ray {leaves/nr:5.2f}  binary reach/ray {rc.sum()/nr:6.2f}  SA(internal)/SA(root) {sa:7.1f}")

if 0: nodes, r = lbvh(); evaluate(nodes, r, "lbvh")
if 0: nodes, r = sah(); evaluate(nodes, r, "sah32")

def evaluate_dp(nodes, root, label, Cv=1.0, Ct=0.15):
    nn = len(nodes)
    child = np.array(nodes, dtype=np.int64)
    blo = np.zeros((nn, 3)); bhi = np.zeros((nn, 3))
    order = [root]
    for n in order:
        for c in child[n]:
            if c >= 0: order.append(c)
    def cbox(c):
        return (tlo[~c], thi[~c]) if c < 0 else (blo[c], bhi[c])
    for n in order[::-1]:
        l, r = cbox(child[n, 0]), cbox(child[n, 1])
        blo[n] = np.minimum(l[0], r[0]); bhi[n] = np.maximum(l[1], r[1])
    def A(c):
        lo, hi = cbox(c); e = np.maximum(hi - lo, 0); return e[0]*e[1]+e[1]*e[2]+e[2]*e[0]
    # f[c][k]: min cost to represent subtree c by exactly k members (k=1..4); rec[c]: cost of a record at c
    INF = float('inf')
    f = {}; rec = {}; choice = {}
    for n in order[::-1]:
        for c in child[n]:
            if c < 0:
                f[c] = [INF, A(c) * Ct, INF, INF, INF]
        L, R = int(child[n, 0]), int(child[n, 1])
        # expanded: k >= 2 from children
        g = [INF] * 5; gc = [None] * 5
        for k1 in range(1, 4):
            for k2 in range(1, 4):
                if k1 + k2 <= 4:
                    v = f[L][k1] + f[R][k2]
                    if v < g[k1 + k2]: g[k1 + k2] = v; gc[k1 + k2] = (k1, k2)
        best = min(range(2, 5), key=lambda k: g[k])
        rec[n] = A(n) * Cv + g[best]
        choice[n] = (best, gc)
        f[n] = [INF, rec[n], g[2], g[3], g[4]]  # as 1 member: its own record; k members: expanded
    # collect records and their cuts
    def members(c, k, gcs):
        if k == 1: return [c]
        k1, k2 = gcs[c][k]
        return members(int(child[c, 0]), k1, gcs) + members(int(child[c, 1]), k2, gcs)
    gcs = {n: choice[n][1] for n in order}
    recs = [root]; cuts = {}
    i = 0
    while i < len(recs):
        n = recs[i]; i += 1
        k = choice[n][0]
        cut = members(n, k, gcs)
        cuts[n] = cut
        recs += [c for c in cut if c >= 0]
    O = S.astype(np.float64); D = E.astype(np.float64) - O
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = 1.0 / D
    def enters(lo, hi):
        t0 = (lo[:, None] - O[None]) * inv[None]; t1 = (hi[:, None] - O[None]) * inv[None]
        t0 = np.where(np.isnan(t0), -np.inf, t0); t1 = np.where(np.isnan(t1), np.inf, t1)
        return np.maximum(np.minimum(t0, t1).max(-1), 0) <= np.minimum(np.maximum(t0, t1).min(-1), 1)
    ent = enters(blo, bhi)
    # reach in the 4-wide tree: record reached iff its node box entered and its parent record reached
    reachr = {root: ent[root]}
    vis = 0; tests = 0
    for n in recs:
        v = reachr[n]; vis += v.sum(); tests += v.sum() * len(cuts[n])
        for c in cuts[n]:
            if c >= 0: reachr[c] = v & ent[c]
    print(f"{label:8s} DP-4 visits/ray {vis/nr:6.2f}  box tests/ray {tests/nr:6.2f}  mean width {np.mean([len(cuts[n]) for n in recs]):.2f}")


Ci, Ct = 1.2, 1.0
def restructure(nodes, root, TL=7, passes=2, minleaves=1):
    child = [list(x) for x in nodes]
    nn = len(child)
    for it in range(passes):
        # boxes, parents, subtree leaf counts, costs
        blo = np.zeros((nn, 3)); bhi = np.zeros((nn, 3)); parent = {}
        order = [root]
        for n in order:
            for c in child[n]:
                parent[c] = n
                if c >= 0: order.append(c)
        def cbox(c): return (tlo[~c], thi[~c]) if c < 0 else (blo[c], bhi[c])
        def A(lo, hi): e = np.maximum(hi - lo, 0); return e[0]*e[1]+e[1]*e[2]+e[2]*e[0]
        cost = {}
        for n in order[::-1]:
            l, r = cbox(child[n][0]), cbox(child[n][1])
            blo[n] = np.minimum(l[0], r[0]); bhi[n] = np.maximum(l[1], r[1])
        def ccost(c): return A(*cbox(c)) * Ct if c < 0 else cost[c]
        for n in order[::-1]:
            cost[n] = A(blo[n], bhi[n]) * Ci + ccost(child[n][0]) + ccost(child[n][1])
        # bottom-up: process nodes in reverse BFS order (children before parents)
        improved = 0
        for n in order[::-1]:
            # form treelet
            tl = list(child[n]); internal_used = []
            while len(tl) < TL:
                cand = [c for c in tl if c >= 0]
                if not cand: break
                c = max(cand, key=lambda c: A(blo[c], bhi[c]))
                tl.remove(c); internal_used.append(c); tl += list(child[c])
            k = len(tl)
            if k < 3: continue
            lo = np.array([cbox(c)[0] for c in tl]); hi = np.array([cbox(c)[1] for c in tl])
            lc = [ccost(c) for c in tl]
            full = (1 << k) - 1
            area = np.zeros(full + 1); copt = np.zeros(full + 1); popt = [0] * (full + 1)
            for s in range(1, full + 1):
                m = [(s >> i) & 1 for i in range(k)]
                idx = [i for i in range(k) if m[i]]
                area[s] = A(lo[idx].min(0), hi[idx].max(0))
            for s in range(1, full + 1):
                if s & (s - 1) == 0:
                    copt[s] = lc[s.bit_length() - 1]; continue
                best = np.inf; bp = 0
                # enumerate proper subsets p of s with lowest bit of s in p (avoid symmetric)
                low = s & -s
                p = (s - 1) & s
                while p:
                    if p & low:
                        v = copt[p] + copt[s ^ p]
                        if v < best: best = v; bp = p
                    p = (p - 1) & s
                copt[s] = area[s] * Ci + best; popt[s] = bp
            if copt[full] < cost[n] - 1e-12:
                improved += 1
                # rebuild treelet topology reusing internal node ids (n root + internal_used)
                free = list(internal_used)
                def make(s):
                    if s & (s - 1) == 0: return tl[s.bit_length() - 1]
                    p = popt[s]
                    node = free.pop() if s != full else n
                    L = make(p); R = make(s ^ p)
                    child[node] = [L, R]
                    return node
                # need to assign root first
                p = popt[full]; L = make(p); R = make(full ^ p); child[n] = [L, R]
                # update boxes/costs for changed nodes: recompute bottom-up locally (simple: recompute all later)
                def upd(c):
                    if c < 0: return
                    upd(child[c][0]); upd(child[c][1])
                    l, r = cbox(child[c][0]), cbox(child[c][1])
                    blo[c] = np.minimum(l[0], r[0]); bhi[c] = np.maximum(l[1], r[1])
                    cost[c] = A(blo[c], bhi[c]) * Ci + ccost(child[c][0]) + ccost(child[c][1])
                # only treelet internal nodes changed; their leaves keep boxes
                def upd_tl(c):
                    if c < 0 or c in tl: return
                    upd_tl(child[c][0]); upd_tl(child[c][1])
                    l, r = cbox(child[c][0]), cbox(child[c][1])
                    blo[c] = np.minimum(l[0], r[0]); bhi[c] = np.maximum(l[1], r[1])
                    cost[c] = A(blo[c], bhi[c]) * Ci + ccost(child[c][0]) + ccost(child[c][1])
                upd_tl(n)
        print(f"pass {it}: improved {improved} treelets, root cost {cost[root]:.4g}", flush=True)
    return [tuple(x) for x in child], root

# ---- hybrid trees: SAH over the top down to subsets of <= S_top
# triangles with the Morton/Karras topology inside them, or the Karras topology
# with every subtree of <= S_bot leaves rebuilt by binned SAH
_lo_all, _hi_all = tlo.min(0), thi.max(0)
_W = (_hi_all - _lo_all).max()
_w = np.maximum(_hi_all - _lo_all, _W / 64)
_q = np.clip(np.floor((cen - _lo_all) / _w * 1024), 0, 1023).astype(np.uint64)
code = expand10(_q[:, 2]) | (expand10(_q[:, 1]) << 1) | (expand10(_q[:, 0]) << 2)
def area(lo, hi):
    e = np.maximum(hi - lo, 0); return e[..., 0]*e[..., 1] + e[..., 1]*e[..., 2] + e[..., 2]*e[..., 0]
def build_sahtop(S_top, nbins=32, mode="sah_top"):
    nodes = []
    def lb(idx):  # Karras over idx sorted by code
        o = idx[np.argsort(code[idx], kind="stable")]; cs = code[o]
        def rec(i, j):
            if i == j: return ~int(o[i])
            if cs[i] == cs[j]: m = (i + j) // 2
            else:
                x = int(cs[i]) ^ int(cs[j]); b = x.bit_length() - 1
                lo_, hi_ = i, j
                while hi_ - lo_ > 1:
                    mid = (lo_ + hi_) // 2
                    if (int(cs[mid]) >> b) == (int(cs[i]) >> b): lo_ = mid
                    else: hi_ = mid
                m = lo_
            k = len(nodes); nodes.append(None); nodes[k] = (rec(i, m), rec(m + 1, j)); return k
        return rec(0, len(o) - 1)
    def sah(idx):
        if len(idx) == 1: return ~int(idx[0])
        if mode == "sah_top" and len(idx) <= S_top: return lb(idx)
        c = cen[idx]; clo, chi = c.min(0), c.max(0); best = (np.inf, None)
        for ax in range(3):
            if chi[ax] - clo[ax] <= 0: continue
            b = np.minimum(((c[:, ax] - clo[ax]) / (chi[ax] - clo[ax]) * nbins).astype(int), nbins - 1)
            blo = np.full((nbins, 3), np.inf); bhi = np.full((nbins, 3), -np.inf); cnt = np.zeros(nbins)
            for k in range(nbins):
                m = b == k
                if m.any(): blo[k] = tlo[idx[m]].min(0); bhi[k] = thi[idx[m]].max(0); cnt[k] = m.sum()
            plo = np.minimum.accumulate(blo); phi = np.maximum.accumulate(bhi); pc = np.cumsum(cnt)
            slo = np.minimum.accumulate(blo[::-1])[::-1]; shi = np.maximum.accumulate(bhi[::-1])[::-1]; sc = np.cumsum(cnt[::-1])[::-1]
            for k in range(nbins - 1):
                if pc[k] == 0 or sc[k + 1] == 0: continue
                cost = area(plo[k], phi[k]) * pc[k] + area(slo[k + 1], shi[k + 1]) * sc[k + 1]
                if cost < best[0]: best = (cost, (ax, b, k))
        if best[1] is None: m = len(idx) // 2; L, R = idx[:m], idx[m:]
        else: ax, b, k = best[1]; L, R = idx[b <= k], idx[b > k]
        kk = len(nodes); nodes.append(None); nodes[kk] = (sah(L), sah(R)); return kk
    return nodes, sah(np.arange(N))
def build_lbtop(S_bot, nbins=32, S_min=1, one_axis=False):
    # Karras over everything; a subtree with <= S_bot leaves is rebuilt by binned SAH,
    # down to S_min leaves (smaller sets: Karras splits of their Morton codes again)
    o = np.argsort(code, kind="stable"); cs = code[o]; nodes = []
    def karras_set(idx):  # idx in Morton order
        if len(idx) == 1: return ~int(idx[0])
        c = code[idx]
        if c[0] == c[-1]: m = len(idx) // 2
        else:
            b = (int(c[0]) ^ int(c[-1])).bit_length() - 1
            m = int(np.argmax((c >> np.uint64(b)) != (c[0] >> np.uint64(b))))
        kk = len(nodes); nodes.append(None); nodes[kk] = (karras_set(idx[:m]), karras_set(idx[m:])); return kk
    def sahb(idx):
        if len(idx) == 1: return ~int(idx[0])
        if len(idx) <= S_min: return karras_set(idx)
        c = cen[idx]; clo, chi = c.min(0), c.max(0); best = (np.inf, None)
        axes = [int(np.argmax(chi - clo))] if one_axis else range(3)
        for ax in axes:
            if chi[ax] - clo[ax] <= 0: continue
            b = np.minimum(((c[:, ax] - clo[ax]) / (chi[ax] - clo[ax]) * nbins).astype(int), nbins - 1)
            blo = np.full((nbins, 3), np.inf); bhi = np.full((nbins, 3), -np.inf); cnt = np.zeros(nbins)
            for k in range(nbins):
                m = b == k
                if m.any(): blo[k] = tlo[idx[m]].min(0); bhi[k] = thi[idx[m]].max(0); cnt[k] = m.sum()
            plo = np.minimum.accumulate(blo); phi = np.maximum.accumulate(bhi); pc = np.cumsum(cnt)
            slo = np.minimum.accumulate(blo[::-1])[::-1]; shi = np.maximum.accumulate(bhi[::-1])[::-1]; sc = np.cumsum(cnt[::-1])[::-1]
            for k in range(nbins - 1):
                if pc[k] == 0 or sc[k + 1] == 0: continue
                cost = area(plo[k], phi[k]) * pc[k] + area(slo[k + 1], shi[k + 1]) * sc[k + 1]
                if cost < best[0]: best = (cost, (ax, b, k))
        if best[1] is None: m = len(idx) // 2; L, R = idx[:m], idx[m:]
        else: ax, b, k = best[1]; L, R = idx[b <= k], idx[b > k]
        kk = len(nodes); nodes.append(None); nodes[kk] = (sahb(L), sahb(R)); return kk
    def rec(i, j):
        if i == j: return ~int(o[i])
        if j - i + 1 <= S_bot: return sahb(o[i:j + 1])
        if cs[i] == cs[j]: m = (i + j) // 2
        else:
            x = int(cs[i]) ^ int(cs[j]); b = x.bit_length() - 1
            lo_, hi_ = i, j
            while hi_ - lo_ > 1:
                mid = (lo_ + hi_) // 2
                if (int(cs[mid]) >> b) == (int(cs[i]) >> b): lo_ = mid
                else: hi_ = mid
            m = lo_
        k = len(nodes); nodes.append(None); nodes[k] = (rec(i, m), rec(m + 1, j)); return k
    return nodes, rec(0, N - 1)

def build_sahtop_sub(S_bot, nbins=10, top_bins=10):
    # the Karras tree's maximal subtrees of <= S_bot leaves (items), each rebuilt by
    # binned SAH (as build_lbtop), and a binned SAH tree over the items' boxes
    # replacing the Karras nodes above them
    o = np.argsort(code, kind="stable"); cs = code[o]
    sub_nodes, _ = [], None
    lb_nodes, lb_root = build_lbtop(S_bot, nbins)
    # items: recompute Karras ranges to find maximal <= S_bot ranges
    items = []
    def rec(i, j):
        if j - i + 1 <= S_bot: items.append((i, j)); return
        if cs[i] == cs[j]: m = (i + j) // 2
        else:
            x = int(cs[i]) ^ int(cs[j]); b = x.bit_length() - 1
            lo_, hi_ = i, j
            while hi_ - lo_ > 1:
                mid = (lo_ + hi_) // 2
                if (int(cs[mid]) >> b) == (int(cs[i]) >> b): lo_ = mid
                else: hi_ = mid
            m = lo_
        rec(i, m); rec(m + 1, j)
    rec(0, N - 1)
    # rebuild: nodes list; each item subtree via SAH (reuse build_lbtop's inner builder by a fresh call on the item's prims)
    nodes = []
    def sah_prims(idx):
        if len(idx) == 1: return ~int(idx[0])
        c = cen[idx]; clo, chi = c.min(0), c.max(0); best = (np.inf, None)
        for ax in range(3):
            if chi[ax] - clo[ax] <= 0: continue
            b = np.minimum(((c[:, ax] - clo[ax]) / (chi[ax] - clo[ax]) * nbins).astype(int), nbins - 1)
            blo = np.full((nbins, 3), np.inf); bhi = np.full((nbins, 3), -np.inf); cnt = np.zeros(nbins)
            for k in range(nbins):
                m = b == k
                if m.any(): blo[k] = tlo[idx[m]].min(0); bhi[k] = thi[idx[m]].max(0); cnt[k] = m.sum()
            plo = np.minimum.accumulate(blo); phi = np.maximum.accumulate(bhi); pc = np.cumsum(cnt)
            slo = np.minimum.accumulate(blo[::-1])[::-1]; shi = np.maximum.accumulate(bhi[::-1])[::-1]; sc = np.cumsum(cnt[::-1])[::-1]
            for k in range(nbins - 1):
                if pc[k] == 0 or sc[k + 1] == 0: continue
                cost = area(plo[k], phi[k]) * pc[k] + area(slo[k + 1], shi[k + 1]) * sc[k + 1]
                if cost < best[0]: best = (cost, (ax, b, k))
        if best[1] is None: m = len(idx) // 2; L, R = idx[:m], idx[m:]
        else: ax, b, k = best[1]; L, R = idx[b <= k], idx[b > k]
        kk = len(nodes); nodes.append(None); nodes[kk] = (sah_prims(L), sah_prims(R)); return kk
    it_ref, it_lo, it_hi = [], [], []
    for (i, j) in items:
        idx = o[i:j + 1]
        it_ref.append(sah_prims(idx)); it_lo.append(tlo[idx].min(0)); it_hi.append(thi[idx].max(0))
    it_lo, it_hi = np.array(it_lo), np.array(it_hi); it_c = (it_lo + it_hi) / 2
    def sah_items(ii):
        if len(ii) == 1: return it_ref[ii[0]]
        c = it_c[ii]; clo, chi = c.min(0), c.max(0); best = (np.inf, None)
        for ax in range(3):
            if chi[ax] - clo[ax] <= 0: continue
            b = np.minimum(((c[:, ax] - clo[ax]) / (chi[ax] - clo[ax]) * top_bins).astype(int), top_bins - 1)
            for k in range(top_bins - 1):
                L, R = b <= k, b > k
                if not L.any() or not R.any(): continue
                cost = area(it_lo[ii][L].min(0), it_hi[ii][L].max(0)) * L.sum() + area(it_lo[ii][R].min(0), it_hi[ii][R].max(0)) * R.sum()
                if cost < best[0]: best = (cost, (ax, b, k))
        if best[1] is None: m = len(ii) // 2; L, R = ii[:m], ii[m:]
        else: ax, b, k = best[1]; L, R = ii[b <= k], ii[b > k]
        kk = len(nodes); nodes.append(None); nodes[kk] = (sah_items(L), sah_items(R)); return kk
    root = sah_items(np.arange(len(items)))
    return nodes, root

nodes, r = lbvh()
t = time.time()
evaluate(nodes, r, "lbvh")
TL = int(sys.argv[2]) if len(sys.argv) > 2 else 7
P = int(sys.argv[3]) if len(sys.argv) > 3 else 2
nodes2, r2 = restructure(nodes, r, TL=TL, passes=P)
print("time", time.time() - t)
evaluate(nodes2, r2, f"trbvh{TL}")
