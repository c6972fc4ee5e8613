"""BVH diagnostics: decode, text dump and Graphviz DOT.

The paper's debugging strategy: copy the tree from the device to
the host, decode every node and inspect connectivity; case study 2 read the
failure off the dump (half-filled "atomic: 1" nodes, untouched nodes, a root
that was never set).  `rsi_bvh_download` provides the arrays and
`rsi_validate` checks the invariants on the GPU; this module turns a download
into the paper's text format (`display_node_contents`) and
into DOT (`bvh_graphviz` -> `bvh_structure.gv`: internal nodes
labelled "[a,b]" with their leaf range, leaves as boxes labelled "[c] d" with
leaf slot c and triangle id d).

Host-side formatting only; node references are printed as typed indices
(`3(L-internal)`) instead of the paper's raw device addresses.
"""
from __future__ import annotations

import numpy as np


def _box_union(b):
    """b: [2, 6] child slots (xlo ylo zlo xhi yhi zhi) -> [6] union."""
    return np.concatenate([np.minimum(b[0, :3], b[1, :3]), np.maximum(b[0, 3:], b[1, 3:])])


def leaf_ranges(d: dict) -> np.ndarray:
    """[n_nodes, 2] first/last leaf slot under each internal node (iterative post-order)."""
    child = d["child"]
    nn = child.shape[0]
    rng = np.full((nn, 2), -1, np.int64)
    if d["n_triangles"] == 1:
        rng[0] = (0, 0)
        return rng
    root = int(d.get("root", 0))
    if root < 0:  # the construction never reached the root (fault injection)
        return rng
    seen = np.zeros(nn, bool)
    stack = [(root, False)]
    while stack:
        i, done = stack.pop()
        if done:
            lo, hi = [], []
            for c in child[i]:
                if c < 0:
                    lo.append(~c)
                    hi.append(~c)
                else:
                    lo.append(rng[c, 0])
                    hi.append(rng[c, 1])
            rng[i] = (min(lo), max(hi))
        elif not seen[i]:  # (a broken tree may repeat or cycle)
            seen[i] = True
            stack.append((i, True))
            stack.extend((int(c), False) for c in child[i] if 0 <= c < nn)
    return rng


def _fmt_box(b):
    return f"x:[{b[0]:.6g},{b[3]:.6g}], y:[{b[1]:.6g},{b[4]:.6g}], z:[{b[2]:.6g},{b[5]:.6g}]"


def dump_text(d: dict) -> str:
    """The paper's node listing for a `rsi_bvh_download` dict."""
    child, box, parent, arr = d["child"], d["box"], d["parent"], d["arrivals"]
    nn, nt = child.shape[0], d["n_triangles"]
    rng = leaf_ranges(d)
    root = int(d.get("root", 0))
    out = ["BVH tree structure", "---------------------------", "Internal nodes"]
    for i in range(nn):
        kinds = ["leaf" if c < 0 else "internal" for c in child[i]]
        refs = [(~c if c < 0 else c) for c in child[i]]
        tag = "  ------ ROOT NODE" if i == root else ""
        par = "" if parent[i] < 0 else str(parent[i] >> 1)
        out.append(f"[{i}] {_fmt_box(_box_union(box[i]))}{tag}")
        out.append(f"self: {i}, parent: {par}")
        out.append(f"indices: {i}(self), {refs[0]}(L-{kinds[0]}), {refs[1]}(R-{kinds[1]})")
        out.append(f"atomic: {arr[i]}, rangeL: {rng[i, 0]}, rangeR: {rng[i, 1]}")
        out.append("")
    sent = int(d.get("sentinel", -1))
    if sent >= 0:  # Apetrei numbering: node N_t - 1 only points at the root
        out.append(f"[{sent}] x:[0,0], y:[0,0], z:[0,0]")
        out.append(f"self: {sent}, parent: ")
        out.append(f"indices: {sent}(self), {root}(L-internal), 0(R-internal)")
        out.append("atomic: 0, rangeL: 0, rangeR: -1")
        out.append("")
    out += ["---------------------------", "Leaf nodes"]
    slot_box = {}
    for i in range(nn):
        for side in range(2):
            if child[i, side] < 0 and np.isfinite(box[i, side, 0]):
                slot_box.setdefault(int(~child[i, side]), box[i, side])
    for k in range(nt):
        b = slot_box.get(k)
        out.append(f"[{k}] " + (_fmt_box(b) if b is not None else "x:[?], y:[?], z:[?]"))
        out.append(f"self: {k}, parent: {parent[nn + k] >> 1}")
        out.append(f"triangleID: {d['leaf_tri'][k]}")
        out.append("")
    return "\n".join(out)


def to_dot(d: dict) -> str:
    """Graphviz DOT of the tree: internal "[a,b]", leaves "[c] d"."""
    child = d["child"]
    nn = child.shape[0]
    rng = leaf_ranges(d)
    lines = ["digraph bvh_structure {", "  node [fontname=Helvetica];"]
    for i in range(nn):
        lines.append(f'  n{i} [shape=ellipse, label="[{rng[i, 0]},{rng[i, 1]}]"];')
    seen = set()
    for i in range(nn):
        for side, c in enumerate(child[i]):
            if c < 0 and not np.isfinite(d["box"][i, side, 0]):
                continue  # the empty right slot of a one-triangle tree
            if c < 0:
                k = int(~c)
                if k not in seen:
                    seen.add(k)
                    lines.append(f'  l{k} [shape=box, label="[{k}] {d["leaf_tri"][k]}"];')
                lines.append(f"  n{i} -> l{k};")
            else:
                lines.append(f"  n{i} -> n{int(c)};")
    lines.append("}")
    return "\n".join(lines) + "\n"
