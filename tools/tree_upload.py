"""Tree-quality experiment on the GPU (one-off, quoted in DESIGN.md 7): trees
built on the HOST by other methods (binned SAH, SAH over the top + LBVH below,
LBVH + larger treelets; tools/treelet_model.py) are uploaded with
rsi_bvh_upload and walked by the same kernels as the default build, so the
query time of a better tree is MEASURED instead of modelled.

  python tools/tree_upload.py prep   (CPU: build the trees -> tools/_data/trees_<wl>.npz)
  python tools/tree_upload.py run    (GPU box: default build vs each uploaded tree, all modes;
                                      outputs must be identical -- a BVH only prunes)
env: WL (sphere), N (1e7 rays), TREES (names to build in prep)."""
import os, sys, time, json
import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
wl = os.environ.get("WL", "sphere")
DATA = os.path.join(ROOT, "tools", "_data")
path = os.path.join(DATA, f"trees_{wl}.npz")


def model_namespace():
    src = open(os.path.join(ROOT, "tools", "treelet_model.py")).read().split("\nnodes, r = lbvh()")[0]
    g = {"__file__": os.path.join(ROOT, "tools", "treelet_model.py")}
    argv, sys.argv = sys.argv, ["x", wl]
    exec(compile(src, "treelet_model", "exec"), g)
    sys.argv = argv
    return g


def to_gpu_layout(nodes, root, V, T):
    """(left, right) refs (>= 0 internal, < 0 ~primitive) -> rsi_bvh_upload arrays:
    internal nodes renumbered breadth-first from the root (node 0), leaf slots in
    depth-first order, fp32 child boxes = exact min/max of the fp32 vertices."""
    order, idx = [root], {root: 0}
    for n in order:
        for c in nodes[n]:
            if c >= 0:
                idx[c] = len(order)
                order.append(c)
    nn = len(order)
    slot, leaf_tri = {}, []

    def dfs(n):  # depth-first leaf order (left first)
        for c in nodes[n]:
            if c < 0:
                slot[~c] = len(leaf_tri)
                leaf_tri.append(~c)
            else:
                dfs(c)
    sys.setrecursionlimit(1000000)
    dfs(root)
    tv = V[T]  # [N, 3, 3] fp32
    tlo, thi = tv.min(1), tv.max(1)
    child = np.zeros((nn, 2), np.int32)
    lo = np.zeros((nn, 3), np.float32)
    hi = np.zeros((nn, 3), np.float32)
    box = np.zeros((nn, 2, 6), np.float32)
    for n in order[::-1]:
        k = idx[n]
        for s, c in enumerate(nodes[n]):
            if c < 0:
                child[k, s] = ~slot[~c]
                b = (tlo[~c], thi[~c])
            else:
                child[k, s] = idx[c]
                b = (lo[idx[c]], hi[idx[c]])
            box[k, s, :3], box[k, s, 3:] = b
        lo[k] = np.minimum(box[k, 0, :3], box[k, 1, :3])
        hi[k] = np.maximum(box[k, 0, 3:], box[k, 1, 3:])
    return child, box, np.asarray(leaf_tri, np.int32)


def prep():
    import synth
    g = model_namespace()
    V, T, _, _, _ = synth.workload(wl, 16, seed=3)
    trees = {}
    want = os.environ.get("TREES", "sah32 sahtop16 lbtop512 trbvh7x3").split()
    for name in want:
        t0 = time.time()
        if name == "sah32":
            nodes, r = g["sah"](32)
        elif name.startswith("sahtopsub"):
            nodes, r = g["build_sahtop_sub"](int(name[9:]))
        elif name.startswith("sahtop"):
            nodes, r = g["build_sahtop"](int(name[6:]))
        elif name.startswith("lbtop"):
            nodes, r = g["build_lbtop"](int(name[5:]))
        elif name == "trbvh7x3":
            n0, r0 = g["lbvh"]()
            nodes, r = g["restructure"](n0, r0, TL=7, passes=3)
        else:
            raise SystemExit(f"unknown tree {name}")
        c, b, lt = to_gpu_layout([tuple(int(x) for x in nd) for nd in nodes], r, V, T)
        trees[f"{name}_child"], trees[f"{name}_box"], trees[f"{name}_leaf"] = c, b, lt
        print(name, "built in", round(time.time() - t0, 1), "s", flush=True)
    os.makedirs(DATA, exist_ok=True)
    np.savez(path, names=np.array(want), **trees)


def run():
    import torch
    import synth
    from paper_2305_01867_b200 import rsi
    n = int(os.environ.get("N", "10000000"))
    V, T, S, E, _ = synth.workload(wl, n, seed=3)
    dev = torch.device("cuda:0")
    Vd, Td, Sd, Ed = (torch.from_numpy(a).to(dev) for a in (V, T, S, E))
    z = np.load(path)
    res = {}

    def timed(h, label):
        outs = {}
        for mode in ("boolean", "barycentric", "intercept_count"):
            out = rsi.alloc_outputs(n, mode, dev)
            for _ in range(2):
                rsi.rsi_intersect(h, Sd, Ed, mode, out=out)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                rsi.rsi_intersect(h, Sd, Ed, mode, out=out)
            e1.record()
            torch.cuda.synchronize()
            res[f"{label}:{mode}"] = round(e0.elapsed_time(e1) / 5, 4)
            outs[mode] = {k: v.cpu().numpy() for k, v in out.items()}
        return outs

    def work(h, label):
        for mode in ("boolean", "barycentric", "intercept_count"):
            rsi.rsi_reset_stats(h)
            rsi.rsi_intersect(h, Sd, Ed, mode)
            st = rsi.rsi_get_stats(h)
            res[f"{label}:{mode}:box_per_ray"] = round(st["box_tests"] / n, 3)

    base = rsi.rsi_build(Vd, Td)
    ref = timed(base, "default")
    hc = rsi.rsi_build(Vd, Td, rsi.Options(counters=True))
    work(hc, "default")
    for name in [str(x) for x in z["names"]]:
        for h, lab in ((base, name), (hc, name)):
            rsi.rsi_bvh_upload(h, z[f"{name}_child"], z[f"{name}_box"], z[f"{name}_leaf"], 0)
        got = timed(base, name)
        work(hc, name)
        same = all(np.array_equal(got[m][k], ref[m][k], equal_nan=True) for m in got for k in got[m])
        res[f"{name}:identical_outputs"] = bool(same)
    for k, v in res.items():
        print(k, json.dumps(v))


if __name__ == "__main__":
    {"prep": prep, "run": run}[sys.argv[1]]()
