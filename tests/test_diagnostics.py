"""-m "not gpu": the BVH dump / DOT formatting (host logic) on the Fig. 3 tree.

The tree is the Karras tree of the Fig. 3 fixture written down by hand: leaves
in Morton order (T0, T3, T1, T2) with the leaf boxes printed at P:332-346,
root 0 splitting [0,1] | [2,3]."""
import numpy as np

from paper_2305_01867_b200 import diagnostics


def fixture_tree(golden):
    g = golden("fig3_case_study1.txt")
    leaves = g["leaf"]
    lb = np.array([[float(x) for x in r[2:]] for r in leaves], np.float32)  # xlo xhi ylo yhi zlo zhi
    box6 = lambda b: np.array([b[0], b[2], b[4], b[1], b[3], b[5]], np.float32)  # noqa: E731
    child = np.array([[1, 2], [~0, ~1], [~2, ~3]], np.int32)
    box = np.zeros((3, 2, 6), np.float32)
    box[1, 0], box[1, 1] = box6(lb[0]), box6(lb[1])
    box[2, 0], box[2, 1] = box6(lb[2]), box6(lb[3])
    box[0, 0] = np.concatenate([np.minimum(box[1, 0, :3], box[1, 1, :3]), np.maximum(box[1, 0, 3:], box[1, 1, 3:])])
    box[0, 1] = np.concatenate([np.minimum(box[2, 0, :3], box[2, 1, :3]), np.maximum(box[2, 0, 3:], box[2, 1, 3:])])
    parent = np.array([-1, 0 << 1 | 0, 0 << 1 | 1, 1 << 1 | 0, 1 << 1 | 1, 2 << 1 | 0, 2 << 1 | 1], np.int32)
    return {"child": child, "box": box, "parent": parent, "arrivals": np.array([2, 2, 2], np.uint32),
            "leaf_tri": np.array([int(r[1]) for r in leaves], np.int32), "n_triangles": 4, "n_nodes": 3}


def test_dot_labels_follow_the_paper(golden):
    """internal "[a,b]" leaf ranges, leaves "[c] d" (slot, triangle)."""
    dot = diagnostics.to_dot(fixture_tree(golden))
    assert dot.startswith("digraph")
    for lab in ("[0,3]", "[0,1]", "[2,3]", "[0] 0", "[1] 3", "[2] 1", "[3] 2"):
        assert f'label="{lab}"' in dot
    assert dot.count("->") == 6


def test_text_dump_reproduces_printed_fields(golden):
    """root over leaves [0,3] with box x:[12,13] y:[2,3] z:[1,1.3];
    leaf boxes and triangle ids in Morton order."""
    txt = diagnostics.dump_text(fixture_tree(golden))
    assert "[0] x:[12,13], y:[2,3], z:[1,1.3]  ------ ROOT NODE" in txt
    assert "atomic: 2, rangeL: 0, rangeR: 3" in txt
    assert "[1] x:[12,13], y:[2,3], z:[1,1.2]" in txt           # the [0,1] subtree
    assert "[2] x:[12,13], y:[2,3], z:[1.1,1.3]" in txt         # the [2,3] subtree
    assert "triangleID: 3" in txt and txt.index("triangleID: 0") < txt.index("triangleID: 3")
    assert "[1] x:[12,12.5], y:[2,3], z:[1,1.2]" in txt         # leaf 1 = T3


def test_leaf_ranges_one_triangle():
    d = {"child": np.array([[~0, ~0]], np.int32), "box": np.full((1, 2, 6), np.inf, np.float32),
         "parent": np.array([-1, 0], np.int32), "arrivals": np.array([2], np.uint32),
         "leaf_tri": np.array([0], np.int32), "n_triangles": 1, "n_nodes": 1}
    d["box"][0, 0] = [0, 0, 0, 1, 1, 0]
    assert diagnostics.leaf_ranges(d).tolist() == [[0, 0]]
    dot = diagnostics.to_dot(d)
    assert dot.count("->") == 1 and 'label="[0] 0"' in dot


def apetrei_fixture_tree(golden):
    """The same tree in the paper's own numbering (golden 'apetrei'
    rows): root = node 1, sentinel = node 3."""
    g = golden("fig3_case_study1.txt")
    base = fixture_tree(golden)
    rows = {int(r[0]): r for r in g["apetrei"]}
    child = np.zeros((3, 2), np.int32)
    for i in range(3):
        r = rows[i]
        child[i] = [int(r[2]) if r[1] == "internal" else ~int(r[2]), int(r[4]) if r[3] == "internal" else ~int(r[4])]
    # Karras node k -> paper node: 0 (root) -> 1, 1 ([0,1]) -> 0, 2 ([2,3]) -> 2
    box = np.stack([base["box"][1], base["box"][0], base["box"][2]])
    parent = np.array([1 << 1 | 0, -1, 1 << 1 | 1, 0 << 1 | 0, 0 << 1 | 1, 2 << 1 | 0, 2 << 1 | 1], np.int32)
    return {**base, "child": child, "box": box, "parent": parent, "root": 1, "sentinel": 3}


def test_apetrei_numbering_dump(golden):
    """NEXT-1 host formatting: the dump in the paper's numbering reproduces the
    printed indices, ranges, root tag and sentinel of P:304-328."""
    g = golden("fig3_case_study1.txt")
    d = apetrei_fixture_tree(golden)
    rng = diagnostics.leaf_ranges(d)
    for r in g["apetrei"]:
        i = int(r[0])
        if i < 3:
            assert rng[i].tolist() == [int(r[6]), int(r[7])]
    txt = diagnostics.dump_text(d)
    assert "[1] x:[12,13], y:[2,3], z:[1,1.3]  ------ ROOT NODE" in txt
    assert "indices: 0(self), 0(L-leaf), 1(R-leaf)" in txt
    assert "indices: 1(self), 0(L-internal), 2(R-internal)" in txt
    assert "indices: 3(self), 1(L-internal), 0(R-internal)" in txt
    assert "atomic: 0, rangeL: 0, rangeR: -1" in txt
    dot = diagnostics.to_dot(d)
    for lab in ("[0,3]", "[0,1]", "[2,3]", "[0] 0", "[1] 3", "[2] 1", "[3] 2"):
        assert f'label="{lab}"' in dot
