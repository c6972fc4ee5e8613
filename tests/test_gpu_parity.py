"""-m gpu: the CUDA path (through the C-ABI) against the CPU oracle, element by element.

Bar (BASELINE.json north_star): boolean, intercept_count
and nearest-triangle index bit-exact on EVERY ray (flagged rays are counted and
reported, never excused); t within 1e-5, dist within 1e-5*|d|, point within
1e-5*max(|O|_inf, |E|_inf).
"""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

DEV = "cuda:0"


@pytest.fixture(scope="module")
def rsi():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2305_01867_b200 import _build, rsi as _rsi
    _build.build_library()
    return _rsi


def to_dev(*arrs):
    return [torch.from_numpy(np.ascontiguousarray(a)).to(DEV) for a in arrs]


def run_all(rsi, V, T, S, E, options=None):
    Vd, Td, Sd, Ed = to_dev(V, T, S, E)
    h = rsi.rsi_build(Vd, Td, options)
    out = {"hit": rsi.rsi_intersect(h, Sd, Ed, "boolean")["hit"].cpu().numpy()}
    b = rsi.rsi_intersect(h, Sd, Ed, "barycentric")
    out.update({k: v.cpu().numpy() for k, v in b.items()})
    out["count"] = rsi.rsi_intersect(h, Sd, Ed, "intercept_count")["count"].cpu().numpy()
    out["stats"] = rsi.rsi_get_stats(h)
    h.free()
    return out


def assert_parity(got, ref, S, E, label=""):
    n_flag = int((ref["flags"] != 0).sum()) if "flags" in ref else 0
    bad_hit = np.nonzero(got["hit"] != ref["hit"])[0]
    bad_cnt = np.nonzero(got["count"] != ref["count"])[0]
    bad_tri = np.nonzero(got["tri"] != ref["tri"])[0]
    assert bad_hit.size == 0, f"{label} boolean mismatches at {bad_hit[:10]} (flagged rays: {n_flag})"
    assert bad_cnt.size == 0, (f"{label} count mismatches at {bad_cnt[:10]}: got {got['count'][bad_cnt[:10]]} "
                               f"ref {ref['count'][bad_cnt[:10]]}")
    assert bad_tri.size == 0, f"{label} tri mismatches at {bad_tri[:10]}"
    m = ref["tri"] >= 0
    d = (E.astype(np.float64) - S)
    dn = np.linalg.norm(d, axis=1)
    assert np.all(np.abs(got["t"][m] - ref["t"][m]) <= 1e-5), label
    assert np.all(np.abs(got["dist"][m] - ref["dist"][m]) <= 1e-5 * np.maximum(dn[m], 1e-30)), label
    scale = np.maximum(np.abs(S).max(1), np.abs(E).max(1))[m]
    assert np.all(np.abs(got["point"][m] - ref["point"][m]).max(1) <= 1e-5 * np.maximum(scale, 1e-30)), label
    assert np.all(np.isnan(got["t"][~m])) and np.all(np.isnan(got["point"][~m]))
    return n_flag


# ------------------------------------------------------------------ paper worked example

def test_fig3_fixture_all_modes(rsi, golden):
    g = golden("fig3_case_study1.txt")
    V, T = synth.fixture()
    S, E = synth.fixture_rays()
    got = run_all(rsi, V, T, S, E)
    assert got["hit"].tolist() == [int(x) for x in g["boolean"][0]]
    for row in g["hit"]:
        i, tri = int(row[0]), int(row[1])
        assert got["tri"][i] == tri
        np.testing.assert_allclose(got["point"][i], np.array(row[2:], float), atol=1e-4)
    ref = oracle.run(V, T, S, E)
    assert_parity(got, ref, S, E, "fig3")


def test_canopy_counts(rsi, golden):
    g = golden("canopy_counts.txt")
    V, T = synth.canopy()
    S, E = synth.fixture_rays()
    got = run_all(rsi, V, T, S, E)
    assert got["count"].tolist() == [int(x) for x in g["count"][0]]


def test_fig3_bvh_structure(rsi, golden):
    """Leaf order (T0, T3, T1, T2) and node boxes of the P:306-346 dump; the
    root splits leaves [0,1] | [2,3] (z-major Morton, reading R8)."""
    g = golden("fig3_case_study1.txt")
    V, T = synth.fixture()
    Vd, Td = to_dev(V, T)
    h = rsi.rsi_build(Vd, Td, rsi.Options(plain_tree=True))  # the Karras topology as built
    d = rsi.rsi_bvh_download(h)
    h.free()
    leaves = g["leaf"]
    assert d["leaf_tri"].tolist() == [int(r[1]) for r in leaves]
    # leaf boxes: the child slot that holds each leaf
    for node in range(d["n_nodes"]):
        for side in range(2):
            ref = d["child"][node, side]
            if ref < 0:
                slot = ~ref
                row = leaves[slot]
                exp = np.array(row[2:], np.float32)  # xlo xhi ylo yhi zlo zhi
                b = d["box"][node, side]             # xlo ylo zlo xhi yhi zhi
                np.testing.assert_allclose([b[0], b[3], b[1], b[4], b[2], b[5]], exp, atol=1e-6)
    # the root's two children are the subtrees [0,1] and [2,3] with the printed boxes
    nodes = {(int(r[0]), int(r[1])): np.array(r[2:], np.float32) for r in g["node"]}
    root = d["child"][0]
    assert root[0] >= 0 and root[1] >= 0
    for side, rng in ((0, (0, 1)), (1, (2, 3))):
        b = d["box"][0, side]
        np.testing.assert_allclose([b[0], b[3], b[1], b[4], b[2], b[5]], nodes[rng], atol=1e-6)
    np.testing.assert_allclose(d["scene_lo"] + d["scene_hi"], [12, 2, 1, 13, 3, 1.3], atol=1e-6)
    assert (d["arrivals"] == 2).all()


# ------------------------------------------------------------------ configs at oracle sizes

def test_config0_unit_cube_all_modes(rsi):
    V, T, S, E, _ = synth.workload("cube", 10_000)
    ref = oracle.run(V, T, S, E)
    got = run_all(rsi, V, T, S, E)
    assert_parity(got, ref, S, E, "cube")


def test_cube_axis_aligned_closed_form(rsi):
    V, T = synth.cube()
    xs = np.linspace(0.0, 1.0, 9)
    pts = [(x, y) for x in xs for y in xs]
    S = np.array([(x, y, -1.0) for x, y in pts], np.float32)
    E = np.array([(x, y, 2.0) for x, y in pts], np.float32)
    ref = oracle.run(V, T, S, E)
    got = run_all(rsi, V, T, S, E)
    assert_parity(got, ref, S, E, "cube-axis")
    inner = np.array([0 < x < 1 and 0 < y < 1 for x, y in pts])
    assert (got["count"][inner] == 2).all()
    np.testing.assert_allclose(got["t"][inner], 1 / 3, atol=1e-7)


@pytest.mark.parametrize("n_rays", [1, 31, 20_011])
def test_sphere_all_modes(rsi, n_rays):
    V, T, S, E, _ = synth.workload("sphere", n_rays)
    ref = oracle.run(V, T, S, E)
    got = run_all(rsi, V, T, S, E)
    assert_parity(got, ref, S, E, "sphere")


@pytest.mark.parametrize("scale,shift", [(1e-20, 0.0), (1e-3, 0.0), (1.0, 3e4), (1e3, -1e6), (1e20, 1e21)])
def test_scaled_translated_scenes(rsi, scale, shift):
    """The 4-wide walk's folded slab (s*inv exact, slack ~ max|pm| |inv|) at
    extreme mesh scales and offsets, with short, unit and very long segments:
    decisions stay those of the oracle (the slab test only has to stay
    conservative, the exact tests decide)."""
    V, T, S, E, _ = synth.workload("sphere", 6000, seed=11)
    rng = np.random.default_rng(11)
    d = E - S
    f = np.float32(10.0) ** rng.integers(-6, 7, size=(len(S), 1)).astype(np.float32)
    E = (S + d * f).astype(np.float32)  # segment lengths from 1e-6 to 1e6 x
    V = (V.astype(np.float64) * scale + shift).astype(np.float32)
    S = (S.astype(np.float64) * scale + shift).astype(np.float32)
    E = (E.astype(np.float64) * scale + shift).astype(np.float32)
    ref = oracle.run(V, T, S, E)
    got = run_all(rsi, V, T, S, E)
    assert_parity(got, ref, S, E, f"scale={scale},shift={shift}")
    assert got["hit"].sum() > 100


def test_folded_terrain_intercept_count(rsi):
    V, T, S, E, _ = synth.workload("terrain", 6000)
    ref = oracle.run(V, T, S, E)
    got = run_all(rsi, V, T, S, E)
    assert_parity(got, ref, S, E, "terrain")
    assert (got["count"] == 3).sum() > 100


def test_paper_terrain_vertical_and_oblique(rsi):
    V, T = synth.paper_terrain()
    S1, E1 = synth.vertical_rays(3000, V, 6)
    lo, hi = V.min(0), V.max(0)
    S2, E2 = synth.box_rays(3000, lo - [0, 0, 5], hi + [0, 0, 5], 8)
    S, E = np.vstack([S1, S2]), np.vstack([E1, E2])
    ref = oracle.run(V, T, S, E)
    got = run_all(rsi, V, T, S, E)
    assert_parity(got, ref, S, E, "paper-terrain")


def test_rays_through_vertices_and_edges_exact(rsi):
    """Adversarial: exactly vertical segments through grid vertices and edge
    midpoints of the paper-scale terrain (coordinates ~1e3).  Every decision
    sits on a triangle boundary; results must still equal the oracle's."""
    V, T = synth.paper_terrain(40, 30)
    rng = np.random.default_rng(5)
    idx = rng.integers(0, len(V) - 1, 800)
    P = V[idx].astype(np.float64)
    Q = V[rng.integers(0, len(V), 800)].astype(np.float64)
    mid = (P[:400] + V[idx[:400] + 1]) / 2  # (mostly) edge midpoints
    P = np.vstack([P, mid])
    S = np.column_stack([P[:, :2], np.full(len(P), 80.0)]).astype(np.float32)
    E = np.column_stack([P[:, :2], np.full(len(P), 40.0)]).astype(np.float32)
    # plus oblique segments aimed at vertices
    S2 = (Q + rng.normal(size=Q.shape) * [30, 30, 10]).astype(np.float32)
    E2 = (2 * Q - S2).astype(np.float32)
    S, E = np.vstack([S, S2]), np.vstack([E, E2])
    ref = oracle.run(V, T, S, E)
    got = run_all(rsi, V, T, S, E)
    n_flag = assert_parity(got, ref, S, E, "vertices")
    assert n_flag > 500  # the case really is on the boundaries


def test_fp64_moller_option_identical(rsi):
    V, T, S, E, _ = synth.workload("sphere", 4000, seed=21)
    a = run_all(rsi, V, T, S, E)
    b = run_all(rsi, V, T, S, E, rsi.Options(fp64_moller=True))
    for k in ("hit", "count", "tri"):
        assert (a[k] == b[k]).all()
    ref = oracle.run(V, T, S, E)
    assert_parity(b, ref, S, E, "fp64")
    assert b["stats"]["fp64_pairs"] == 0  # the fp64 path does not count "uncertain" pairs


# ------------------------------------------------------------------ edge cases

def test_single_triangle_and_degenerates(rsi):
    V = np.float32([[0, 0, 0], [1, 0, 0], [0, 1, 0]])
    T = np.int32([[0, 1, 2]])
    S = np.float32([[0.2, 0.2, 1], [0.9, 0.9, 1], [0.2, 0.2, 0], [0.3, 0.3, 5], [np.nan, 0, 1], [0.2, 0.2, 1]])
    E = np.float32([[0.2, 0.2, -1], [0.9, 0.9, -1], [0.2, 0.2, 0], [0.3, 0.3, 0], [0.1, 0.1, -1], [0.2, 0.2, 0]])
    ref = oracle.run(V, T, S, E)
    got = run_all(rsi, V, T, S, E)
    assert_parity(got, ref, S, E, "single")
    assert got["hit"].tolist() == [1, 0, 0, 1, 0, 1]
    assert got["stats"]["nonfinite_rays"] >= 1


def test_stacked_identical_triangles_and_overflow_repass(rsi):
    """30 coincident copies + 20 parallel sheets: duplicate Morton codes
    (index-augmented delta), nearest-tie -> lowest id, and > 8 hits per ray
    (register-list overflow -> exact re-pass)."""
    base = np.float32([[0, 0, 0], [1, 0, 0], [0, 1, 0]])
    Vs, Ts = [], []
    for k in range(30):
        Vs.append(base + [0, 0, 0.5]); Ts.append(np.arange(3) + 3 * len(Ts))
    for k in range(20):
        Vs.append(base + [0, 0, 1.0 + 0.01 * k]); Ts.append(np.arange(3) + 3 * len(Ts))
    V = np.vstack(Vs).astype(np.float32)
    T = np.vstack(Ts).astype(np.int32)
    S, E = synth.box_rays(3000, [-0.2, -0.2, -1], [1.2, 1.2, 2.5], 9)
    S[:500, 2] = -1
    E[:500, 2] = 3
    E[:500, :2] = S[:500, :2]
    ref = oracle.run(V, T, S, E)
    Vd, Td, Sd, Ed = to_dev(V, T, S, E)
    h = rsi.rsi_build(Vd, Td)
    got = run_all(rsi, V, T, S, E)
    assert_parity(got, ref, S, E, "stacked")
    assert (got["count"] >= 9).sum() > 50
    d = rsi.rsi_bvh_download(h)
    assert sorted(d["leaf_tri"].tolist()) == list(range(len(T)))
    assert (d["arrivals"] == 2).all()
    h.free()


def test_deferred_build_status(rsi):
    """RSI_OPT_DEFERRED_STATUS: rsi_build/rsi_rebuild return at once, the
    device-side input checks surface in rsi_build_status (and in calls that
    read the build back); valid meshes give the same results as a checked build."""
    V, T = synth.fixture()
    Vd, Td = to_dev(V, T)
    opt = rsi.Options(deferred_status=True)
    bad = torch.tensor([[0, 1, 9]], dtype=torch.int32, device=DEV)
    h = rsi.rsi_build(Vd, bad, opt)  # no error yet
    with pytest.raises(rsi.RsiError) as e:
        rsi.rsi_build_status(h)
    assert e.value.status == 3
    with pytest.raises(rsi.RsiError):  # the handle holds no mesh after the failed check
        rsi.rsi_intersect(h, Vd[:1], Vd[1:2], "boolean")
    rsi.rsi_rebuild(h, Vd, Td)
    rsi.rsi_build_status(h)
    Vn = V.copy()
    Vn[2, 1] = np.nan
    rsi.rsi_rebuild(h, to_dev(Vn)[0], Td)
    with pytest.raises(rsi.RsiError) as e:
        rsi.rsi_bvh_info(h)
    assert e.value.status == 4
    h.free()
    V, T, S, E, _ = synth.workload("sphere", 5000, seed=21)
    Vd, Td, Sd, Ed = to_dev(V, T, S, E)
    ref = oracle.run(V, T, S, E)
    h = rsi.rsi_build(Vd, Td, opt)
    for mode, key in (("boolean", "hit"), ("intercept_count", "count"), ("barycentric", "tri")):
        for _ in range(2):  # rebuild + query back to back, no host read-back
            rsi.rsi_rebuild(h, Vd, Td)
            got = rsi.rsi_intersect(h, Sd, Ed, mode)[key].cpu().numpy()
        assert (got == ref[key]).all(), mode
    rsi.rsi_build_status(h)
    assert rsi.rsi_validate(h)["ok"]
    h.free()


def test_build_errors(rsi):
    V, T = synth.fixture()
    Vd, Td = to_dev(V, T)
    with pytest.raises(rsi.RsiError) as e:
        rsi.rsi_build(Vd, torch.tensor([[0, 1, 9]], dtype=torch.int32, device=DEV))
    assert e.value.status == 3
    Vn = V.copy()
    Vn[2, 1] = np.nan
    with pytest.raises(rsi.RsiError) as e:
        rsi.rsi_build(to_dev(Vn)[0], Td)
    assert e.value.status == 4
    with pytest.raises(rsi.RsiError) as e:
        rsi.rsi_build(Vd, torch.zeros((0, 3), dtype=torch.int32, device=DEV))
    assert e.value.status == 2
    with pytest.raises(TypeError):
        rsi.rsi_build(Vd, Td.long())
    h = rsi.rsi_build(Vd, Td)
    z = torch.zeros((0, 3), dtype=torch.float32, device=DEV)
    assert rsi.rsi_intersect(h, z, z, "boolean")["hit"].numel() == 0
    h.free()


@pytest.mark.parametrize("nt", [1, 2, 3, 17, 1000, 10_240, 16_384, 16_385, 70_001, -5000, "dup"])
def test_bvh_integrity_random_meshes(rsi, nt):
    """Validator invariants (P:407-464 failure signatures must be absent):
    leaf bijection, arrivals == 2, root reachable from every leaf, child boxes
    exact unions, parent/child links mutual; sorted Morton codes equal a
    bit-loop z-major encoding of the fp32 centroids, in stable order (sizes
    span the rank sort, N_t <= 16384, and the radix paths; "dup" repeats 40
    triangles 12000 times, so equal keys must keep index order)."""
    dup = nt == "dup"
    flat = not dup and nt < 0  # a flat (terrain-like) mesh: z extent 1/1000 of x, y
    nt = 12_000 if dup else abs(nt)
    rng = np.random.default_rng(nt)
    V = rng.uniform(-3, 7, (3 * nt, 3)).astype(np.float32)
    if flat:
        V[:, 2] *= np.float32(1e-3)
    T = rng.permutation(3 * nt).reshape(nt, 3).astype(np.int32)
    if dup:
        T = T[:40][rng.integers(0, 40, nt)]
    Vd, Td = to_dev(V, T)
    h = rsi.rsi_build(Vd, Td, rsi.Options(plain_tree=True))  # the Karras tree over the sorted codes
    d = rsi.rsi_bvh_download(h)
    h.free()
    # morton reference (bit loop) on fp32 centroids
    lo, hi = V.min(0), V.max(0)
    c = (V[T[:, 0]] + V[T[:, 1]] + V[T[:, 2]]) / np.float32(3)
    w = np.maximum(hi - lo, (hi - lo).max() * np.float32(1 / 64))   # reading R8: extent floor
    q = np.clip(np.floor((c - lo) / w * np.float32(1024)), 0, 1023).astype(np.uint32)
    code = np.zeros(nt, np.uint32)
    for b in range(10):
        for a in range(3):
            code |= ((q[:, a] >> b) & 1) << (3 * b + a)
    order = np.argsort(code, kind="stable")
    assert (d["morton"] == code[order]).all()
    assert (d["leaf_tri"] == order).all()
    _check_tree(d, V, T, nt, contiguous=True)
    # the default build (SAH-rebuilt subtrees + treelets over the same codes): the same invariants
    h = rsi.rsi_build(Vd, Td)
    d = rsi.rsi_bvh_download(h)
    h.free()
    assert (d["morton"] == code[order]).all()
    _check_tree(d, V, T, nt)


def _check_tree(d, V, T, nt, contiguous=False):
    """Leaf bijection, arrivals == 2, mutual parent / child links, child boxes
    equal to the exact unions; `contiguous`: every node over a contiguous range
    of leaf slots with its id at one end of it (the Karras numbering)."""
    nn = d["n_nodes"]
    assert sorted(d["leaf_tri"].tolist()) == list(range(nt))
    assert (d["arrivals"] == 2).all()
    if nt == 1:
        return
    # boxes: recompute bottom-up and compare exactly
    tb = np.concatenate([V[T].min(1), V[T].max(1)], 1)  # per original triangle
    box, rng = {}, {}

    def node_box(ref):
        if ref < 0:
            return tb[d["leaf_tri"][~ref]]
        if ref in box:
            return box[ref]
        raise KeyError

    def node_rng(ref):
        return (~ref, ~ref) if ref < 0 else rng[ref]

    parent = d["parent"]
    assert parent[0] == -1
    for i in range(nn):
        for side in range(2):
            ch = d["child"][i, side]
            p = parent[ch] if ch >= 0 else parent[nn + ~ch]
            assert p == (i << 1 | side)
    # iterative post-order
    stack = [(0, False)]
    while stack:
        i, done = stack.pop()
        if done:
            l, r = (node_box(x) for x in d["child"][i])
            exp = [np.concatenate([np.minimum(l[:3], r[:3]), np.maximum(l[3:], r[3:])])]
            got_l, got_r = d["box"][i]
            assert (got_l == l).all() and (got_r == r).all()
            box[i] = exp[0]
            if contiguous:
                (a0, a1), (b0, b1) = (node_rng(x) for x in d["child"][i])
                assert a1 + 1 == b0, (i, a0, a1, b0, b1)
                rng[i] = (a0, b1)
                assert i in (a0, b1)
        else:
            stack.append((i, True))
            for ch in d["child"][i]:
                if ch >= 0:
                    stack.append((int(ch), False))
    assert len(box) == nn


def test_compaction_and_sparse_return(rsi):
    V, T, S, E, _ = synth.workload("sphere", 50_000, seed=13)
    Vd, Td, Sd, Ed = to_dev(V, T, S, E)
    h = rsi.rsi_build(Vd, Td)
    out = rsi.rsi_intersect(h, Sd, Ed, "barycentric")
    ids, dist, tri, pts = rsi.sparse_barycentric(out)
    dense = {k: v.cpu().numpy() for k, v in out.items()}
    exp = np.nonzero(dense["tri"] >= 0)[0]
    assert (ids.cpu().numpy() == exp).all()
    # rsi_gather_hits: the hit rows, bit for bit
    assert (tri.cpu().numpy() == dense["tri"][exp]).all()
    assert (dist.cpu().numpy().view(np.uint32) == dense["dist"][exp].view(np.uint32)).all()
    assert (pts.cpu().numpy().view(np.uint32) == dense["point"][exp].view(np.uint32)).all()
    h.free()


def test_rsi_test_host_end_to_end(rsi):
    """The paper's user call on host arrays through rsi_test."""
    V, T, S, E, _ = synth.workload("sphere", 5000, seed=17)
    ref = oracle.run(V, T, S, E)
    b = rsi.rsi_test(V, T, S, E, {"mode": "boolean"})
    assert b.shape == (5000, 1) and (b[:, 0] == ref["hit"].astype(bool)).all()
    c = rsi.rsi_test(V, T, S, E, {"mode": "intercept_count"})
    assert (c == ref["count"]).all()
    ids, dist, tri, pts = rsi.rsi_test(V, T, S, E, {"mode": "barycentric"})
    rids, rdist, rtri, rpts = oracle.sparse_barycentric(ref)
    assert (ids == rids).all() and (tri == rtri).all()
    np.testing.assert_allclose(pts, rpts, atol=1e-5 * 1.5)


# ------------------------------------------------------------------ full sizes (sampled)

def test_bench_size_sampled_parity(rsi):
    """configs[2]-size: N_t = 1e4, N_r = 1e7 in the launch configuration the
    bench times; a seeded sample of 2000 rays is checked against the oracle one
    by one, and mode consistency is checked on all 1e7 rays."""
    V, T, S, E, _ = synth.workload("sphere", 10_000_000, seed=3)
    Vd, Td, Sd, Ed = to_dev(V, T, S, E)
    h = rsi.rsi_build(Vd, Td)
    hit = rsi.rsi_intersect(h, Sd, Ed, "boolean")["hit"].cpu().numpy()
    bar = {k: v.cpu().numpy() for k, v in rsi.rsi_intersect(h, Sd, Ed, "barycentric").items()}
    cnt = rsi.rsi_intersect(h, Sd, Ed, "intercept_count")["count"].cpu().numpy()
    h.free()
    assert ((bar["tri"] >= 0) == (hit > 0)).all()
    assert ((cnt > 0) == (hit > 0)).all()
    rng = np.random.default_rng(0)
    sample = np.sort(rng.choice(len(S), 2000, replace=False))
    ref = oracle.run(V, T, S[sample], E[sample])
    got = {"hit": hit[sample], "count": cnt[sample], **{k: v[sample] for k, v in bar.items()}}
    assert_parity(got, ref, S[sample], E[sample], "1e7-sample")


def test_million_triangle_mesh_sampled(rsi):
    """configs[4] mesh (N_t = 1e6, multi-block radix sort, 6.8% duplicate
    codes): 1e6 rays, 64 sampled against the oracle."""
    V, T, S, E, _ = synth.workload("sphere1m", 1_000_000)
    Vd, Td, Sd, Ed = to_dev(V, T, S, E)
    h = rsi.rsi_build(Vd, Td)
    d = rsi.rsi_bvh_download(h)
    assert (d["arrivals"] == 2).all()
    assert (np.bincount(d["leaf_tri"], minlength=len(T)) == 1).all()
    hit = rsi.rsi_intersect(h, Sd, Ed, "boolean")["hit"].cpu().numpy()
    bar = {k: v.cpu().numpy() for k, v in rsi.rsi_intersect(h, Sd, Ed, "barycentric").items()}
    cnt = rsi.rsi_intersect(h, Sd, Ed, "intercept_count")["count"].cpu().numpy()
    h.free()
    sample = np.arange(0, len(S), len(S) // 64)[:64]
    ref = oracle.run(V, T, S[sample], E[sample], flags=False)
    got = {"hit": hit[sample], "count": cnt[sample], **{k: v[sample] for k, v in bar.items()}}
    assert_parity(got, ref, S[sample], E[sample], "1m-sample")


# ------------------------------------------------------------------ NEXT-2: validator, dump, fault injection

def test_validator_accepts_built_trees(rsi):
    for nt in (1, 2, 5, 1000, 29260, 70001):
        rng = np.random.default_rng(nt)
        V = rng.uniform(-1, 1, (3 * nt, 3)).astype(np.float32)
        T = np.arange(3 * nt, dtype=np.int32).reshape(nt, 3)
        Vd, Td = to_dev(V, T)
        h = rsi.rsi_build(Vd, Td)
        rep = rsi.rsi_validate(h)
        h.free()
        assert rep["ok"], (nt, rep)


def test_case_study_2_failure_signatures(rsi):
    """the construct kernel launched with grid_lambda = 16 blocks of
    1024 threads instead of grid_dimsT = 29 covered only 16 384 of the 29 260
    leaves of a ~30k-triangle terrain.  Injecting the same under-sized refit
    grid reproduces the signatures the paper read off the dump: half-filled
    nodes ("atomic: 1"), untouched nodes ("atomic: 0") and no root box."""
    V, T = synth.paper_terrain()
    assert len(T) == 29260
    Vd, Td = to_dev(V, T)
    h = rsi.rsi_build(Vd, Td, rsi.Options(debug_refit_leaves=16 * 1024))
    rep = rsi.rsi_validate(h)
    assert not rep["ok"]
    assert rep["half_filled"] > 0 and rep["untouched"] > 0 and rep["root_ok"] == 0
    d = rsi.rsi_bvh_download(h)
    h.free()
    assert (d["arrivals"] == 1).sum() == rep["half_filled"]
    assert (d["arrivals"] == 0).sum() == rep["untouched"]
    from paper_2305_01867_b200 import diagnostics
    assert "atomic: 1," in diagnostics.dump_text(d) and "atomic: 0," in diagnostics.dump_text(d)
    # the correct grid gives a valid tree
    h = rsi.rsi_build(Vd, Td)
    assert rsi.rsi_validate(h)["ok"]
    h.free()


def test_fixture_dump_and_dot_from_device(rsi):
    from paper_2305_01867_b200 import diagnostics
    V, T = synth.fixture()
    Vd, Td = to_dev(V, T)
    h = rsi.rsi_build(Vd, Td, rsi.Options(plain_tree=True))
    d = rsi.rsi_bvh_download(h)
    h.free()
    txt = diagnostics.dump_text(d)
    assert "[0] x:[12,13], y:[2,3], z:[1,1.3]  ------ ROOT NODE" in txt
    assert "atomic: 2, rangeL: 0, rangeR: 3" in txt
    dot = diagnostics.to_dot(d)
    for lab in ("[0,3]", "[0,1]", "[2,3]", "[0] 0", "[1] 3", "[2] 1", "[3] 2"):
        assert f'label="{lab}"' in dot


def test_launch_counter(rsi):
    """rsi_launch_count (the bench's gpu_launches) counts every library kernel:
    one traversal kernel per rsi_intersect without overflow, and a build chain
    of at least init/extent/morton/sort/karras/refit per rsi_build."""
    V, T, S, E, _ = synth.workload("sphere", 2000, seed=3)
    Vd, Td, Sd, Ed = to_dev(V, T, S, E)
    c0 = rsi.rsi_launch_count()
    h = rsi.rsi_build(Vd, Td)
    c1 = rsi.rsi_launch_count()
    assert c1 - c0 >= 6
    for mode in ("boolean", "barycentric", "intercept_count"):
        before = rsi.rsi_launch_count()
        ovf0 = rsi.rsi_get_stats(h)["overflow_rays"]
        rsi.rsi_intersect(h, Sd, Ed, mode)
        # + the re-pass kernels when some segment overflowed the count list
        # (one-traversal pass + dedup; + size / collect / dedup beyond 64 hits)
        launched = rsi.rsi_launch_count() - before
        # intercept_count always enqueues its exact re-pass (no host read-back of the overflow count)
        assert launched == (2 if mode == "intercept_count" else 1), (mode, launched)
    c2 = rsi.rsi_launch_count()
    rsi.rsi_rebuild(h, Vd, Td)
    assert rsi.rsi_launch_count() - c2 == c1 - c0
    h.free()


# ------------------------------------------------------------------ NEXT-1: 63-bit Morton + Apetrei build

def _morton63_ref(V, T):
    """Bit-loop reference of the 63-bit z-major code on fp32 centroids (reading
    R8 scaled to 21 bits per axis)."""
    lo, hi = V.min(0), V.max(0)
    c = (V[T[:, 0]] + V[T[:, 1]] + V[T[:, 2]]) / np.float32(3)
    w = np.maximum(hi - lo, (hi - lo).max() * np.float32(1 / 64))
    q = np.clip(np.floor((c - lo) / w * np.float32(2 ** 21)), 0, 2 ** 21 - 1).astype(np.uint64)
    code = np.zeros(len(T), np.uint64)
    for b in range(21):
        for a in range(3):
            code |= ((q[:, a] >> np.uint64(b)) & np.uint64(1)) << np.uint64(3 * b + a)
    return code


def test_apetrei_fixture_numbering(rsi, golden):
    """The paper's own tree for the Fig. 3 fixture: root = node 1,
    node i splits leaves i | i+1, sentinel 3 -> root, leaf order T0 T3 T1 T2,
    every node reached twice ("atomic: 2")."""
    from paper_2305_01867_b200 import diagnostics
    g = golden("fig3_case_study1.txt")
    V, T = synth.fixture()
    Vd, Td = to_dev(V, T)
    h = rsi.rsi_build(Vd, Td, rsi.Options(apetrei=True))
    d = rsi.rsi_bvh_download(h)
    assert rsi.rsi_validate(h)["ok"]
    h.free()
    assert d["root"] == 1 and d["sentinel"] == 3
    assert d["leaf_tri"].tolist() == [int(r[1]) for r in g["leaf"]]
    for r in g["apetrei"]:
        i = int(r[0])
        if i == 3:
            continue
        exp = [int(r[2]) if r[1] == "internal" else ~int(r[2]), int(r[4]) if r[3] == "internal" else ~int(r[4])]
        assert d["child"][i].tolist() == exp, i
        assert d["arrivals"][i] == int(r[5])
    nodes = {(int(r[0]), int(r[1])): np.array(r[2:], np.float32) for r in g["node"]}
    rng = diagnostics.leaf_ranges(d)
    for i in range(3):
        b = diagnostics._box_union(d["box"][i])
        np.testing.assert_allclose([b[0], b[3], b[1], b[4], b[2], b[5]], nodes[tuple(rng[i])], atol=1e-6)
    assert (d["morton"] == (d["morton63"] >> np.uint64(33)).astype(np.uint32)).all()
    txt = diagnostics.dump_text(d)
    assert "[1] x:[12,13], y:[2,3], z:[1,1.3]  ------ ROOT NODE" in txt
    assert "indices: 3(self), 1(L-internal), 0(R-internal)" in txt


@pytest.mark.parametrize("nt", [2, 3, 17, 1000, 16_384, 16_385, 70_001, "dup", "flat"])
def test_apetrei_tree_integrity(rsi, nt):
    """63-bit codes equal a bit-loop encoding in stable sorted order (rank-sort
    and radix paths, full 32-bit low words); the validator finds no violation;
    node i is the split between leaves i and i+1 (the paper's numbering)."""
    from paper_2305_01867_b200 import diagnostics
    kind = nt if isinstance(nt, str) else ""
    nt = 12_000 if kind else nt
    rng = np.random.default_rng(nt + len(kind))
    V = rng.uniform(-3, 7, (3 * nt, 3)).astype(np.float32)
    if kind == "flat":
        V[:, 2] *= np.float32(1e-3)
    T = rng.permutation(3 * nt).reshape(nt, 3).astype(np.int32)
    if kind == "dup":
        T = T[:40][rng.integers(0, 40, nt)]
    Vd, Td = to_dev(V, T)
    h = rsi.rsi_build(Vd, Td, rsi.Options(apetrei=True))
    rep = rsi.rsi_validate(h)
    d = rsi.rsi_bvh_download(h)
    h.free()
    assert rep["ok"], rep
    code = _morton63_ref(V, T)
    order = np.argsort(code, kind="stable")
    assert (d["morton63"] == code[order]).all()
    assert (d["leaf_tri"] == order).all()
    assert (d["arrivals"] == 2).all() and d["sentinel"] == nt - 1
    lr = diagnostics.leaf_ranges(d)
    assert lr[d["root"]].tolist() == [0, nt - 1]
    for i in range(nt - 1):
        c = d["child"][i]
        left_hi = ~c[0] if c[0] < 0 else lr[c[0], 1]
        right_lo = ~c[1] if c[1] < 0 else lr[c[1], 0]
        assert left_hi == i and right_lo == i + 1


def test_apetrei_parity_all_modes(rsi):
    """Same results as the default build (and the oracle) on the bench mesh,
    the folded terrain and rays through vertices/edges."""
    V, T, S, E, _ = synth.workload("sphere", 20_011, seed=3)
    assert_parity(run_all(rsi, V, T, S, E, rsi.Options(apetrei=True)), oracle.run(V, T, S, E), S, E, "sphere")
    V, T, S, E, _ = synth.workload("terrain", 4_000, seed=4)
    assert_parity(run_all(rsi, V, T, S, E, rsi.Options(apetrei=True)), oracle.run(V, T, S, E), S, E, "terrain")
    V, T = synth.cube()
    S, E = synth.box_rays(5_000, -0.5, 1.5, seed=1)
    assert_parity(run_all(rsi, V, T, S, E, rsi.Options(apetrei=True)), oracle.run(V, T, S, E), S, E, "cube")


def test_apetrei_fault_injection_signatures(rsi):
    """Case study 2 on the paper's construction: an under-sized
    grid leaves half-filled and untouched nodes, leaves not connected to the
    root and no root; every ray then misses (no crash)."""
    V, T = synth.paper_terrain()
    Vd, Td = to_dev(V, T)
    h = rsi.rsi_build(Vd, Td, rsi.Options(apetrei=True, debug_refit_leaves=16 * 1024))
    rep = rsi.rsi_validate(h)
    assert not rep["ok"]
    assert rep["half_filled"] > 0 and rep["untouched"] > 0 and rep["root_ok"] == 0
    assert rep["unreachable_leaves"] > 0
    assert rsi.rsi_bvh_root(h)["root"] == -1
    S, E = synth.vertical_rays(1000, V, seed=4)
    Sd, Ed = to_dev(S, E)
    assert int(rsi.rsi_intersect(h, Sd, Ed, "boolean")["hit"].sum()) == 0
    h.free()


def test_apetrei_sort_full_low_words(rsi):
    """The 63-bit path sorts the low 32 code bits as a full-range key: codes
    whose low word is 0xffffffff (q_x, q_y = ...11111111111, q_z = ...1111111111)
    must still sort stably (the rank sort's k+1 wraps there)."""
    rng = np.random.default_rng(7)
    pts = [np.zeros(3), np.ones(3)]                      # extent [0,1]^3: q = floor(c * 2^21)
    for _ in range(1500):                                # low word all ones, varied high bits
        hx, hy, hz = rng.integers(0, 1024, 3)
        q = np.array([hx * 2048 + 2047, hy * 2048 + 2047, hz * 1024 + 1023], np.float64)
        pts.append((q + 0.5) / 2 ** 21)
    pts += list(rng.uniform(0, 1, (1500, 3)))
    P = np.asarray(pts, np.float32)
    V = np.repeat(P, 3, axis=0)                          # point-like triangles: centroid = the point
    T = np.arange(len(V), dtype=np.int32).reshape(-1, 3)
    T = T[rng.permutation(len(T))]
    Vd, Td = to_dev(V, T)
    h = rsi.rsi_build(Vd, Td, rsi.Options(apetrei=True))
    d = rsi.rsi_bvh_download(h)
    assert rsi.rsi_validate(h)["ok"]
    h.free()
    code = _morton63_ref(V, T)
    assert int(((code & np.uint64(0xffffffff)) == np.uint64(0xffffffff)).sum()) >= 1000
    order = np.argsort(code, kind="stable")
    assert (d["morton63"] == code[order]).all()
    assert (d["leaf_tri"] == order).all()


@pytest.mark.parametrize("n_sheets", [40, 100, 256, 300, 700, 1500, "coincident"])
def test_overflow_warp_dedup(rsi, n_sheets):
    """Rays crossing up to 1500 stacked sheets overflow the 4-entry hit list:
    the re-pass (k_count_repass) takes every hit's fp64 t, one warp per ray
    sorts the keys (t, slot) and counts gaps by ballot; more than 512 hits
    take several windows of 256 keys (700, 1500 sheets), with the last t
    carried across windows.  Sheets come in groups whose members are 1e-7
    apart in z (merged by tau) and groups 0.004 apart (distinct);
    "coincident": 600 copies of one sheet (t ties across a window boundary)
    between distinct sheets.  Counts equal the oracle's exactly."""
    base = np.float32([[-1, -1, 0], [3, -1, 0], [-1, 3, 0]])
    Vs, z = [], 1.0
    if n_sheets == "coincident":
        for k in range(5):
            Vs.append(base + np.float32([0, 0, 1.0 + 0.01 * k]))
        for k in range(600):
            Vs.append(base + np.float32([0, 0, 1.1]))
        for k in range(5):
            Vs.append(base + np.float32([0, 0, 1.2 + 0.01 * k]))
        z = 1.3
    for k in range(n_sheets if isinstance(n_sheets, int) else 0):
        z += 1e-7 if k % 3 else 0.004
        Vs.append(base + np.float32([0, 0, z]))
    V = np.vstack(Vs).astype(np.float32)
    T = np.arange(len(V), dtype=np.int32).reshape(-1, 3)
    rng = np.random.default_rng(n_sheets if isinstance(n_sheets, int) else 7)
    S = np.column_stack([rng.uniform(0, 1, 400), rng.uniform(0, 1, 400), np.full(400, 0.5)]).astype(np.float32)
    E = S.copy()
    E[:, 2] = np.float32(z + 0.5)
    E[:200, :2] += rng.uniform(-0.2, 0.2, (200, 2)).astype(np.float32)  # some oblique
    ref = oracle.run(V, T, S, E)
    got = run_all(rsi, V, T, S, E)
    assert (got["count"] == ref["count"]).all(), np.nonzero(got["count"] != ref["count"])[0][:10]
    assert got["stats"]["overflow_rays"] > 0 and ref["count"].max() > 8


def test_rsi_test_sparse_device_compaction(rsi):
    """rsi_test_sparse (the paper's barycentric return) over several
    1 Mi-ray chunks with a ragged tail: compaction (3a) and gather on
    the device give exactly the dense path's hits in ascending ray order; no
    hits -> empty arrays."""
    V, T, S, E, _ = synth.workload("sphere", 2_500_003, seed=21)
    ids, dist, tri, pts = rsi.rsi_test(V, T, S, E, {"mode": "barycentric"})
    dense = rsi.rsi_test(V, T, S, E, {"mode": "barycentric"}, sparse=False)
    dt = dense["tri"].numpy()
    rid = np.nonzero(dt >= 0)[0]
    assert (ids == rid).all()
    assert (tri == dt[rid]).all()
    assert (dist == dense["dist"].numpy()[rid]).all()
    assert (pts == dense["point"].numpy()[rid]).all()
    sample = rid[:: max(1, len(rid) // 300)][:300]
    ref = oracle.run(V, T, S[sample], E[sample], flags=False)
    assert (ref["tri"] == dt[sample]).all()
    far = S + np.float32(10.0)
    ids0, dist0, tri0, pts0 = rsi.rsi_test(V, T, far[:1000], (E + np.float32(10.0))[:1000], {"mode": "barycentric"})
    assert len(ids0) == len(dist0) == len(tri0) == len(pts0) == 0
    z = np.zeros((0, 3), np.float32)
    assert all(len(a) == 0 for a in rsi.rsi_test(V, T, z, z, {"mode": "barycentric"}))


def test_pycudarsi_call_shape(rsi):
    """`with PyCudaRSI(design_params) as pycu: pycu.test(...)` in every
    mode, with USE_DOUBLE_PRECISION_MOLLER giving identical results."""
    V, T, S, E, _ = synth.workload("cube", 3000, seed=1)
    ref = oracle.run(V, T, S, E)
    for params in ({}, {"USE_DOUBLE_PRECISION_MOLLER": True, "USE_EXTRA_BVH_FIELDS": True}):
        with rsi.PyCudaRSI(params) as pycu:
            b = pycu.test(V, T, S, E, {"mode": "boolean"})
            c = pycu.test(V, T, S, E, {"mode": "intercept_count"})
            ids, dist, tri, pts = pycu.test(V, T, S, E, {"mode": "barycentric"})
        assert (b[:, 0] == ref["hit"].astype(bool)).all() and (c == ref["count"]).all()
        rids, rdist, rtri, rpts = oracle.sparse_barycentric(ref)
        assert (ids == rids).all() and (tri == rtri).all()
        np.testing.assert_allclose(pts, rpts, atol=1e-5 * 2)


def test_rotate_option_parity_and_integrity(rsi):
    """RSI_OPT_ROTATE (local SAH rotations fused into the refit) changes the
    tree, never the results: every mode matches the oracle and the validator
    finds no violation; leaves keep their Morton order."""
    for name, nr in (("sphere", 20_011), ("terrain", 4_000), ("paper_terrain", 3_000)):
        V, T, S, E, _ = synth.workload(name, nr, seed=5)
        assert_parity(run_all(rsi, V, T, S, E, rsi.Options(rotate=True)), oracle.run(V, T, S, E), S, E, name)
    for nt in (2, 3, 1000, 16_385, 70_001):
        rng = np.random.default_rng(nt)
        V = rng.uniform(-3, 7, (3 * nt, 3)).astype(np.float32)
        T = rng.permutation(3 * nt).reshape(nt, 3).astype(np.int32)
        Vd, Td = to_dev(V, T)
        h = rsi.rsi_build(Vd, Td, rsi.Options(rotate=True))
        rep = rsi.rsi_validate(h)
        d = rsi.rsi_bvh_download(h)
        h.free()
        assert rep["ok"], (nt, rep)
        assert sorted(d["leaf_tri"].tolist()) == list(range(nt))


def test_peer_outputs_single_rank(rsi):
    """PeerOutputs (the fused alternative to the gather): the
    traversal writes into rank 0's symmetric buffers through the mapped
    pointer and the device barrier completes the step; on one rank the result
    equals a plain rsi_intersect bit for bit."""
    import os
    import socket
    import torch.distributed as dist
    from paper_2305_01867_b200.sharded import PeerOutputs
    own = not dist.is_initialized()
    if own:
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(sk.getsockname()[1]))
        sk.close()
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device(DEV))
    try:
        V, T, S, E, _ = synth.workload("sphere", 100_003, seed=8)
        Vd, Td, Sd, Ed = to_dev(V, T, S, E)
        h = rsi.rsi_build(Vd, Td)
        for mode in ("boolean", "barycentric", "intercept_count"):
            peer = PeerOutputs(len(S), mode, torch.device(DEV))
            ref = rsi.rsi_intersect(h, Sd, Ed, mode)
            for step in range(3):  # the same buffers reused step after step (begin / complete)
                peer.begin()
                rsi.rsi_intersect(h, Sd, Ed, mode, out=peer.outputs())
                peer.complete()
                torch.cuda.synchronize()
                for k, v in peer.result().items():
                    a, b = v.cpu(), ref[k].cpu()
                    assert torch.equal(a, b) or bool(((a == b) | (torch.isnan(a) & torch.isnan(b))).all()), (mode, k)
                    v.fill_(0)  # the next step must rewrite every row
        h.free()
    finally:
        if own:
            dist.destroy_process_group()


def test_gather_pipeline_nccl_single_rank(rsi):
    """GatherPipeline on the NCCL backend (world size 1 here: the multi-rank run
    needs more GPUs): async device-side gathers into reused receive buffers,
    all three modes, equal to the local outputs."""
    import os
    import socket
    import torch.distributed as dist
    from paper_2305_01867_b200.sharded import FIELDS, GatherPipeline
    own = not dist.is_initialized()
    if own:
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(sk.getsockname()[1]))
        sk.close()
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device(DEV))
    try:
        V, T, S, E, _ = synth.workload("sphere", 50_001, seed=9)
        Vd, Td, Sd, Ed = to_dev(V, T, S, E)
        h = rsi.rsi_build(Vd, Td)
        pipe = GatherPipeline(slots=2)
        for step, mode in enumerate(("boolean", "barycentric", "intercept_count", "barycentric")):
            out = rsi.rsi_intersect(h, Sd, Ed, mode)
            got = pipe.start(step % 2, {f: out[f] for f in FIELDS[mode]}, len(S)).wait()
            torch.cuda.synchronize()
            for k, v in got.items():
                a, b = v.cpu(), out[k].cpu()
                assert torch.equal(a, b) or bool(((a == b) | (torch.isnan(a) & torch.isnan(b))).all()), (mode, k)
        pipe.drain()
        h.free()
    finally:
        if own:
            dist.destroy_process_group()


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_fuzz_degenerate_soups(rsi, seed):
    """Random triangle soups mixing slivers (aspect ~1e6), zero-area triangles
    (collinear / repeated vertices), huge and tiny triangles and coordinates at
    1e4 offsets, against segments that are short, long, axis-aligned, through
    vertices or of zero length: every mode equals the exhaustive oracle on
    every ray (with and without RSI_OPT_ROTATE / RSI_OPT_APETREI)."""
    rng = np.random.default_rng(100 + seed)
    nt = 3000
    base = rng.uniform(-1, 1, (nt, 3))
    kind = rng.integers(0, 5, nt)
    e1 = rng.normal(size=(nt, 3)) * rng.choice([1e-4, 1e-2, 1.0], nt)[:, None]
    e2 = rng.normal(size=(nt, 3)) * rng.choice([1e-4, 1e-2, 1.0], nt)[:, None]
    e2[kind == 1] = e1[kind == 1] * 2.0          # collinear
    e1[kind == 2] = 0.0                          # repeated vertex
    e2[kind == 3] = e1[kind == 3] + rng.normal(size=(int((kind == 3).sum()), 3)) * 1e-6  # sliver
    off = np.float64(1e4 if seed % 2 else 0.0)
    V = np.stack([base, base + e1, base + e2], 1).reshape(-1, 3) + off
    V = V.astype(np.float32)
    T = np.arange(3 * nt, dtype=np.int32).reshape(nt, 3)
    nr = 6000
    S = (rng.uniform(-1.5, 1.5, (nr, 3)) + off).astype(np.float32)
    E = (S + rng.normal(size=(nr, 3)) * rng.choice([0.01, 0.5, 3.0], nr)[:, None]).astype(np.float32)
    k = nr // 6
    E[:k] = S[:k]                                               # zero length
    E[k:2 * k] = S[k:2 * k]
    E[k:2 * k, 2] += np.float32(2.0)                            # axis-aligned
    vi = rng.integers(0, len(V), k)
    S[2 * k:3 * k] = V[vi] - np.float32(0.3)                    # through vertices
    E[2 * k:3 * k] = V[vi] + np.float32(0.3)
    ref = oracle.run(V, T, S, E)
    for opts in (None, rsi.Options(rotate=True), rsi.Options(apetrei=True)):
        assert_parity(run_all(rsi, V, T, S, E, opts), ref, S, E, f"fuzz{seed} {opts}")


def test_dedup_gaps_near_tau(rsi):
    """intercept_count single-linkage decisions right at the threshold: pairs of
    sheets whose crossings differ by 0.5 .. 1.5 tau in t (reading R4), where the
    fp32 path must defer to the fp64 mirror; counts equal the oracle's."""
    base = np.float32([[-2, -2, 0], [4, -2, 0], [-2, 4, 0]])
    # the second sheet of each pair is tilted in x: over the rays' footprint
    # x in [0, 1] the gap to the first runs from 0.5 tau to 1.5 tau
    tilt = np.array([[0, 0, 1e-6 * (0.5 + v[0])] for v in base])
    Vs = []
    z = 0.25
    rng = np.random.default_rng(5)
    for k in range(3):
        Vs.append(base + np.float32([0, 0, z]))
        Vs.append((base.astype(np.float64) + tilt + [0, 0, z]).astype(np.float32))
        z += 0.2
    V = np.vstack(Vs).astype(np.float32)
    T = np.arange(len(V), dtype=np.int32).reshape(-1, 3)
    nr = 20_000
    S = np.column_stack([rng.uniform(0, 1, nr), rng.uniform(0, 1, nr), np.zeros(nr)]).astype(np.float32)
    E = S.copy()
    E[:, 2] = np.float32(1.0)
    E[:, :2] += rng.uniform(-1e-3, 1e-3, (nr, 2)).astype(np.float32)
    ref = oracle.run(V, T, S, E)
    got = run_all(rsi, V, T, S, E)
    assert (got["count"] == ref["count"]).all(), np.nonzero(got["count"] != ref["count"])[0][:10]
    assert len(np.unique(ref["count"])) > 1 and got["stats"]["fp64_rays"] > 0  # both sides of tau occur


def _depth_of_tree(d):
    """Max root-to-leaf depth of a downloaded tree (binary levels)."""
    child, root = d["child"], d["root"]
    depth, best, stack = {root: 0}, 0, [root]
    while stack:
        n = stack.pop()
        for c in child[n]:
            if c >= 0:
                depth[c] = depth[n] + 1
                stack.append(c)
            else:
                best = max(best, depth[n] + 1)
    return best


def test_deep_chain_tree_stack_bound(rsi):
    """A comb of triangles at 2^-i along each axis (i = 1 .. 21) gives Morton codes
    with (nearly) one bit set each: every split peels one triangle off, so the
    tree is a chain (depth 39 with the 63-bit codes of RSI_OPT_APETREI).  Segments through
    the nested boxes near the origin walk the whole chain; with greedy 4-cut
    records a member may sit one level down, so the lane stack needs 3 entries
    per level (kStackQuad = 288 >= 3 x 95).  Every mode equals the oracle."""
    pts = []
    for ax in range(3):
        for i in range(1, 22):
            p = np.zeros(3)
            p[ax] = 2.0 ** -i
            pts.append(p)
    tris = []
    for p in pts:
        s = 0.25 * max(p.max(), 2.0 ** -21)
        tris.append([p + [-s, -s, 0.3 * s], p + [s, -s, -0.3 * s], p + [0, s, 0]])
    tris.append([[0, 0, 0], [1, 1, 1], [1, 0, 1]])   # scene extent [0, 1]^3
    V = np.array(tris, np.float64).reshape(-1, 3).astype(np.float32)
    T = np.arange(len(V), dtype=np.int32).reshape(-1, 3)
    rng = np.random.default_rng(11)
    nr = 8000
    S = rng.uniform(-0.05, 0.05, (nr, 3)).astype(np.float32) * rng.choice([1.0, 1e-3, 1e-5], nr)[:, None].astype(np.float32)
    E = rng.uniform(0.0, 0.6, (nr, 3)).astype(np.float32) * rng.choice([1.0, 1e-2, 1e-4], nr)[:, None].astype(np.float32)
    ref = oracle.run(V, T, S, E)
    assert ref["count"].max() >= 3
    Vd, Td = to_dev(V, T, S, E)[:2]
    for opts in (None, rsi.Options(apetrei=True)):
        h = rsi.rsi_build(Vd, Td, opts)
        depth = _depth_of_tree(rsi.rsi_bvh_download(h))
        h.free()
        assert depth >= (32 if opts is not None else 12), depth  # measured: 39 under RSI_OPT_APETREI
        assert_parity(run_all(rsi, V, T, S, E, opts), ref, S, E, f"chain {opts} depth {depth}")


def _sah_cost(d):
    """Surface-area cost of a downloaded tree: sum of internal-node areas / root area."""
    b = d["box"].astype(np.float64)                           # [nn, 2, 6]
    lo = np.minimum(b[:, 0, :3], b[:, 1, :3])
    hi = np.maximum(b[:, 0, 3:], b[:, 1, 3:])
    e = np.maximum(hi - lo, 0)
    a = e[:, 0] * e[:, 1] + e[:, 1] * e[:, 2] + e[:, 2] * e[:, 0]
    return a.sum() / a[d["root"]]


@pytest.mark.parametrize("wl", ["sphere", "paper_terrain"])
def test_treelet_restructuring_lowers_sah_same_results(rsi, wl):
    """The default build rebuilds completed treelets for least surface-area
    cost (RSI_OPT_PLAIN_TREE keeps the Karras topology): the tree is valid
    (validator), its SAH cost is lower, and every mode's outputs are identical
    to the plain tree's and to the oracle's."""
    V, T, S, E, _ = synth.workload(wl, 20_011, seed=17)
    Vd, Td = to_dev(V, T)
    costs = {}
    for plain in (True, False):
        h = rsi.rsi_build(Vd, Td, rsi.Options(plain_tree=plain))
        assert rsi.rsi_validate(h)["ok"]
        d = rsi.rsi_bvh_download(h)
        h.free()
        assert sorted(d["leaf_tri"].tolist()) == list(range(len(T)))
        costs[plain] = _sah_cost(d)
    assert costs[False] < 0.95 * costs[True], costs
    ref = oracle.run(V, T, S, E)
    a = run_all(rsi, V, T, S, E, rsi.Options(plain_tree=True))
    b = run_all(rsi, V, T, S, E)
    assert_parity(b, ref, S, E, wl)
    for k in ("hit", "count", "tri"):
        assert (a[k] == b[k]).all(), k


def _median_tree(V, T, seed):
    """A valid binary tree that is neither Karras nor SAH: recursive splits at a
    random position of the triangles sorted along a random axis (host, numpy),
    in the rsi_bvh_upload layout (internal nodes breadth-first from 0, leaf
    slots depth-first, fp32 child boxes = exact unions)."""
    rng = np.random.default_rng(seed)
    tv = V[T]
    tlo, thi, cen = tv.min(1), tv.max(1), tv.mean(1)
    nodes = []

    def build(idx):
        if len(idx) == 1:
            return ~int(idx[0])
        ax = int(rng.integers(0, 3))
        idx = idx[np.argsort(cen[idx, ax], kind="stable")]
        m = int(rng.integers(1, len(idx)))
        k = len(nodes)
        nodes.append(None)
        nodes[k] = (build(idx[:m]), build(idx[m:]))
        return k

    import sys
    sys.setrecursionlimit(100000)
    root = build(np.arange(len(T)))
    order, pos = [root], {root: 0}
    for n in order:
        for c in nodes[n]:
            if c >= 0:
                pos[c] = len(order)
                order.append(c)
    slot, leaf_tri = {}, []

    def dfs(n):
        for c in nodes[n]:
            if c < 0:
                slot[~c] = len(leaf_tri)
                leaf_tri.append(~c)
            else:
                dfs(c)

    dfs(root)
    nn = len(order)
    child = np.zeros((nn, 2), np.int32)
    box = np.zeros((nn, 2, 6), np.float32)
    lo, hi = np.zeros((nn, 3), np.float32), np.zeros((nn, 3), np.float32)
    for n in order[::-1]:
        i = pos[n]
        for s, c in enumerate(nodes[n]):
            if c < 0:
                child[i, s], b = ~slot[~c], (tlo[~c], thi[~c])
            else:
                child[i, s], b = pos[c], (lo[pos[c]], hi[pos[c]])
            box[i, s, :3], box[i, s, 3:] = b
        lo[i], hi[i] = np.minimum(box[i, 0, :3], box[i, 1, :3]), np.maximum(box[i, 0, 3:], box[i, 1, 3:])
    return child, box, np.asarray(leaf_tri, np.int32)


@pytest.mark.parametrize("wl", ["sphere", "terrain"])
def test_bvh_upload_any_tree_same_results(rsi, wl):
    """rsi_bvh_upload (the inverse of rsi_bvh_download): a host-built tree of
    random splits replaces the built one; the 4-wide records are rebuilt from it
    and every mode still equals the oracle element by element (the BVH only
    prunes), and a download returns the uploaded topology."""
    V, T, S, E, _ = synth.workload(wl, 20_011, seed=23)
    ref = oracle.run(V, T, S, E)
    child, box, leaf = _median_tree(V, T, 5)
    Vd, Td, Sd, Ed = to_dev(V, T, S, E)
    h = rsi.rsi_build(Vd, Td)
    rsi.rsi_bvh_upload(h, child, box, leaf, 0)
    d = rsi.rsi_bvh_download(h)
    assert (d["child"] == child).all() and (d["box"] == box).all() and (d["leaf_tri"] == leaf).all()
    assert rsi.rsi_validate(h)["ok"]  # parent links, arrivals, root reached from every leaf
    got = {"hit": rsi.rsi_intersect(h, Sd, Ed, "boolean")["hit"].cpu().numpy()}
    got.update({k: v.cpu().numpy() for k, v in rsi.rsi_intersect(h, Sd, Ed, "barycentric").items()})
    got["count"] = rsi.rsi_intersect(h, Sd, Ed, "intercept_count")["count"].cpu().numpy()
    assert_parity(got, ref, S, E, f"upload {wl}")
    with pytest.raises(Exception):
        rsi.rsi_bvh_upload(h, child, box, leaf[::-1].copy() * 0, 0)  # not a permutation
    h.free()


@pytest.mark.parametrize("case", ["outliers", "n63", "n64", "n257", "gate32768", "gate32769", "coincident"])
def test_sah_subtree_build_edge_cases(rsi, case):
    """The default build's SAH subtree pass (N_t <= 32768) and its fused refit on
    trees that stress it: isolated far-away triangles (single leaves and two-leaf
    nodes directly under Karras nodes of > 256 leaves: the leftover items),
    the size gates (no pass below 64 or above 32768 triangles), a whole tree that
    is one subtree (257 is just above), and coincident centroids (every split
    degenerate: median splits).  Every tree is checked by the validator and the
    exact-box walk of _check_tree, and all modes equal the oracle."""
    rng = np.random.default_rng(77)
    nt = {"outliers": 5003, "n63": 63, "n64": 64, "n257": 257, "gate32768": 32768, "gate32769": 32769,
          "coincident": 3000}[case]
    V = rng.uniform(0, 1, (3 * nt, 3)).astype(np.float32)
    if case == "outliers":  # three isolated triangles far from the cluster, one pair close together
        V[-9:] = np.float32([[40, 40, 40], [40.1, 40, 40], [40, 40.1, 40],
                             [-30, 5, 5], [-30, 5.1, 5], [-30, 5, 5.1],
                             [-30.2, 5, 5], [-30.2, 5.1, 5], [-30.2, 5, 5.1]])
    if case == "coincident":  # the same triangle (same centroid) 3000 times, a few distinct ones
        V[3:3 * (nt - 5)] = np.tile(V[:3], (nt - 6, 1))
    T = np.arange(3 * nt, dtype=np.int32).reshape(nt, 3)
    Vd, Td = to_dev(V, T)
    h = rsi.rsi_build(Vd, Td)
    assert rsi.rsi_validate(h)["ok"]
    d = rsi.rsi_bvh_download(h)
    h.free()
    _check_tree(d, V, T, nt)
    if case == "outliers":  # the leftover items exist: a leaf child of a node with > 256 leaves
        child = d["child"]
        size = {}

        def leaves(i):
            if i < 0:
                return 1
            if i not in size:
                size[i] = leaves(int(child[i, 0])) + leaves(int(child[i, 1]))
            return size[i]

        import sys
        sys.setrecursionlimit(100000)
        leaves(0)
        assert any(size[i] > 256 and (child[i] < 0).any() for i in size)
    S, E = synth.box_rays(3000 if nt < 20000 else 800, [-1, -1, -1], [2, 2, 2], 5)
    if case == "outliers":
        S[:20], E[:20] = np.float32([40.03, 40.03, 39]), np.float32([40.03, 40.03, 41])
        S[20:40], E[20:40] = np.float32([-31, 5.02, 5.02]), np.float32([-29, 5.02, 5.02])
    ref = oracle.run(V, T, S, E)
    got = run_all(rsi, V, T, S, E)
    assert_parity(got, ref, S, E, case)
    if case == "outliers":
        assert got["hit"][:20].all() and (got["count"][20:40] == 2).all()


def test_overlapped_steps_two_handles_two_streams(rsi):
    """bench.py's overlapped steps: consecutive rebuild + intersect pairs
    alternate between two handles and two streams with no host sync, so step
    k+1's rebuild runs while step k's traversal is still in flight.  Every
    step's outputs equal the oracle (all modes, every ray)."""
    V, T, S, E, _ = synth.workload("sphere", 60_001, seed=17)
    ref = oracle.run(V, T, S, E)
    Vd, Td, Sd, Ed = to_dev(V, T, S, E)
    hs = [rsi.rsi_build(Vd, Td, rsi.Options(deferred_status=True)) for _ in range(2)]
    sts = [torch.cuda.Stream(), torch.cuda.Stream()]
    modes = ("boolean", "barycentric", "intercept_count")
    outs = [{m: rsi.alloc_outputs(len(S), m, DEV) for m in modes} for _ in range(6)]
    torch.cuda.synchronize()
    for k in range(6):
        with torch.cuda.stream(sts[k % 2]):
            rsi.rsi_rebuild(hs[k % 2], Vd, Td)
            for m in modes:
                rsi.rsi_intersect(hs[k % 2], Sd, Ed, m, out=outs[k][m])
    torch.cuda.synchronize()
    for h in hs:
        rsi.rsi_build_status(h)
        h.free()
    for k in range(6):
        got = {"hit": outs[k]["boolean"]["hit"].cpu().numpy(), "count": outs[k]["intercept_count"]["count"].cpu().numpy()}
        got.update({f: v.cpu().numpy() for f, v in outs[k]["barycentric"].items()})
        assert_parity(got, ref, S, E, f"step {k}")
