"""Pins for the CPU oracle (oracle/rsi_oracle.c) -- all -m "not gpu".

Every check ties the oracle to something other than itself: values printed in
the paper (Fig. 3; canopy P:365), exact-rational plane
clipping (a different algorithm from Moller-Trumbore), the closed-form unit
cube, closed-mesh crossing parity, 2D column counts on a folded terrain, and
brute-force exact arithmetic on tiny random meshes.
"""
from fractions import Fraction as Fr

import numpy as np
import pytest

import oracle
import synth
from referee import brute_force_exact, cube_clip_exact, seg_tri_exact


# ----------------------------------------------------------------- paper worked example

def test_fig3_boolean_tri_and_points(golden):
    """P:351 boolean vector and P:200 hit triangles / points (1e-4 abs)."""
    g = golden("fig3_case_study1.txt")
    V, T = synth.fixture()
    S, E = synth.fixture_rays()
    r = oracle.run(V, T, S, E)
    assert r["hit"].tolist() == [int(x) for x in g["boolean"][0]]
    hits = {int(row[0]): (int(row[1]), np.array(row[2:], float)) for row in g["hit"]}
    for i in range(8):
        if i in hits:
            tri, p = hits[i]
            assert r["tri"][i] == tri
            np.testing.assert_allclose(r["point"][i], p, atol=1e-4)
            # vertical segment from z = 2: distance to the hit = 2 - z
            assert abs(r["dist"][i] - (2.0 - p[2])) < 1e-4
        else:
            assert r["tri"][i] == -1 and np.isnan(r["t"][i])
    assert r["count"].tolist() == r["hit"].tolist()
    assert not r["flags"].any()


def test_canopy_counts(golden):
    """intercept_count on the canopy surface: 2 through a patch + base."""
    g = golden("canopy_counts.txt")
    V, T = synth.canopy()
    S, E = synth.fixture_rays()
    r = oracle.run(V, T, S, E)
    assert r["count"].tolist() == [int(x) for x in g["count"][0]]


# ----------------------------------------------------------------- exact referee

@pytest.mark.parametrize("seed", range(6))
def test_random_tiny_meshes_match_exact_referee(seed):
    rng = np.random.default_rng(100 + seed)
    nt = int(rng.integers(1, 17))
    V = rng.uniform(0, 1, (3 * nt, 3)).astype(np.float32)
    T = np.arange(3 * nt, dtype=np.int32).reshape(nt, 3)
    S, E = synth.box_rays(150, -0.5, 1.5, seed)
    r = oracle.run(V, T, S, E)
    ref = brute_force_exact(V.tolist(), T.tolist(), S.tolist(), E.tolist())
    for i, (h, c, tri, t) in enumerate(ref):
        assert r["hit"][i] == int(h), i
        assert r["count"][i] == c, i
        assert r["tri"][i] == tri, i
        if h:
            assert abs(r["t"][i] - float(t)) <= 1e-12 * max(1.0, abs(float(t)))


def test_near_edge_adversarial_pairs_match_exact_referee():
    """Terrain-scale coordinates (~1e3), triangles ~25 units, points
    placed within ~1e-9 (barycentric) of an edge, segment lengths 10..3000
    (SURVEY A.7).  The double oracle must decide exactly as exact arithmetic."""
    rng = np.random.default_rng(7)
    n_disagree = n_hit = 0
    for k in range(1500):
        A = rng.uniform(900, 1100, 3)
        B = A + rng.uniform(-25, 25, 3)
        C = A + rng.uniform(-25, 25, 3)
        A, B, C = (x.astype(np.float32).astype(np.float64) for x in (A, B, C))
        edge = [(A, B, C), (B, C, A), (C, A, B)][k % 3]
        s = rng.uniform(0, 1)
        off = rng.choice([-1, 1]) * 10.0 ** rng.uniform(-12, -8)
        P = edge[0] + s * (edge[1] - edge[0]) + off * (edge[2] - edge[0])
        d = rng.normal(size=3)
        d *= rng.uniform(10, 3000) / np.linalg.norm(d)
        t0 = rng.uniform(0.05, 0.95)
        O = (P - t0 * d).astype(np.float32)
        Ee = (P + (1 - t0) * d).astype(np.float32)
        h, t, u, v, det = oracle.mt(O, Ee, A, B, C)
        te = seg_tri_exact(O, Ee, A, B, C)
        n_hit += te is not None
        if h != (te is not None):
            n_disagree += 1
        elif h:
            assert abs(t - float(te)) < 1e-9
    assert n_disagree == 0
    assert 200 < n_hit < 1300  # both sides of the edges are exercised


# ----------------------------------------------------------------- closed forms

def test_unit_cube_random_segments_closed_form():
    V, T = synth.cube()
    S, E = synth.box_rays(1500, -0.5, 1.5, 1)
    r = oracle.run(V, T, S, E)
    for i in range(len(S)):
        c, t = cube_clip_exact(S[i], E[i])
        assert r["count"][i] == c, i
        assert r["hit"][i] == int(c > 0)
        if c:
            assert abs(r["t"][i] - float(t)) < 1e-12
            d = E[i].astype(np.float64) - S[i]
            np.testing.assert_allclose(r["point"][i], S[i] + float(t) * d, atol=1e-12)
            assert abs(r["dist"][i] - float(t) * np.linalg.norm(d)) < 1e-12


def test_unit_cube_axis_aligned_families():
    """(x,y,-1)->(x,y,2): count 2, t = 1/3, point (x,y,0), dist 1;
    (x,y,0.5)->(x,y,2): count 1, t = 1/3, dist 0.5."""
    V, T = synth.cube()
    xs = [0.125, 0.25, 0.5, 0.75, 0.875]
    pts = [(x, y) for x in xs for y in xs]
    S1 = np.array([(x, y, -1.0) for x, y in pts], np.float32)
    E1 = np.array([(x, y, 2.0) for x, y in pts], np.float32)
    r = oracle.run(V, T, S1, E1)
    assert (r["count"] == 2).all()
    assert np.allclose(r["t"], 1.0 / 3.0, atol=1e-15)
    assert np.allclose(r["dist"], 1.0, atol=1e-14)
    assert np.allclose(r["point"][:, 2], 0.0, atol=1e-15)
    # points on the face diagonal x == y hit both triangles of the face: 4 raw
    # hits, deduplicated to 2 crossings (single linkage, reading R4)
    diag = np.array([x == y for x, y in pts])
    assert (r["nhits_raw"][diag] == 4).all() and (r["nhits_raw"][~diag] == 2).all()
    S2 = S1.copy()
    S2[:, 2] = 0.5
    r2 = oracle.run(V, T, S2, E1)
    assert (r2["count"] == 1).all()
    assert np.allclose(r2["t"], 1.0 / 3.0, atol=1e-15)
    assert np.allclose(r2["dist"], 0.5, atol=1e-14)


def test_closed_sphere_crossing_parity():
    """Closed mesh: count parity = inside(start) xor inside(end).  Inside:
    |p| < 0.9 (below every facet), outside: |p| > 1.07 (above every vertex)."""
    V, T = synth.uv_sphere()
    S, E = synth.box_rays(20000, -1.5, 1.5, 11)
    rs, re = np.linalg.norm(S, axis=1), np.linalg.norm(E, axis=1)
    ok = ((rs < 0.9) | (rs > 1.07)) & ((re < 0.9) | (re > 1.07))
    S, E = S[ok][:2500], E[ok][:2500]
    r = oracle.run(V, T, S, E)
    inside = lambda p: np.linalg.norm(p, axis=1) < 0.9  # noqa: E731
    assert ((r["count"] % 2) == (inside(S) ^ inside(E))).all()
    assert ((r["count"] > 0) == (r["hit"] > 0)).all()


def test_folded_terrain_vertical_column_counts():
    """Exactly vertical segments spanning the folded sheet: the number of
    crossings equals the number of triangles whose xy projection contains the
    column (a 2D point-in-triangle count, independent of Moller-Trumbore)."""
    V, T = synth.folded_terrain()
    S, E = synth.vertical_rays(400, V, 4, jitter=0.0)
    r = oracle.run(V, T, S, E)
    P = V.astype(np.float64)[T]            # [nt, 3, 3]
    a, b, c = P[:, 0, :2], P[:, 1, :2], P[:, 2, :2]
    checked = 0
    for i in range(len(S)):
        q = S[i, :2].astype(np.float64)
        e0 = (b[:, 0] - a[:, 0]) * (q[1] - a[:, 1]) - (b[:, 1] - a[:, 1]) * (q[0] - a[:, 0])
        e1 = (c[:, 0] - b[:, 0]) * (q[1] - b[:, 1]) - (c[:, 1] - b[:, 1]) * (q[0] - b[:, 0])
        e2 = (a[:, 0] - c[:, 0]) * (q[1] - c[:, 1]) - (a[:, 1] - c[:, 1]) * (q[0] - c[:, 0])
        m = np.minimum(np.abs(e0), np.minimum(np.abs(e1), np.abs(e2)))
        inside = ((e0 > 0) & (e1 > 0) & (e2 > 0)) | ((e0 < 0) & (e1 < 0) & (e2 < 0))
        if (m < 1e-3).any():               # column too close to a projected edge
            continue
        checked += 1
        assert r["count"][i] == int(inside.sum()), i
    assert checked > 300
    assert (r["count"] == 3).any() and (r["count"] == 1).any()


# ----------------------------------------------------------------- invariants & readings

def test_mode_consistency_and_reversal():
    V, T = synth.uv_sphere()
    S, E = synth.box_rays(1500, -1.5, 1.5, 12)
    r = oracle.run(V, T, S, E)
    rr = oracle.run(V, T, E, S)
    assert ((r["count"] > 0) == (r["hit"] > 0)).all()
    assert ((r["tri"] >= 0) == (r["hit"] > 0)).all()
    clean = (r["flags"] == 0) & (rr["flags"] == 0)
    assert (r["hit"][clean] == rr["hit"][clean]).all()
    assert (r["nhits_raw"][clean] == rr["nhits_raw"][clean]).all()
    assert (r["count"][clean] == rr["count"][clean]).all()


def test_nearest_tie_takes_lowest_triangle_id_and_flags_B():
    V, T = synth.fixture()
    T2 = np.vstack([T, T[[1]]]).astype(np.int32)           # duplicate T1 as id 4
    T2 = T2[[0, 4, 2, 3, 1]].astype(np.int32)              # ids: dup at 1, original at 4
    S, E = synth.fixture_rays()
    r = oracle.run(V, T2, S, E)
    assert r["tri"][2] == 1                                 # lower of {1, 4}
    assert r["flags"][2] & oracle.FLAG_B
    assert r["count"][2] == 1 and r["nhits_raw"][2] == 2


def test_flags_edge_touch_parallel_dedup():
    V, T = synth.fixture()
    # through the centre vertex (12.5, 2.5): on all four triangles' corner
    r = oracle.run(V, T, np.float32([[12.5, 2.5, 2.0]]), np.float32([[12.5, 2.5, 0.0]]))
    assert r["flags"][0] & oracle.FLAG_E and r["count"][0] == 1 and r["nhits_raw"][0] == 4
    Vc, Tc = synth.cube()
    # ends exactly on the bottom face: t = 1 -> touch
    r = oracle.run(Vc, Tc, np.float32([[0.3, 0.4, -1.0]]), np.float32([[0.3, 0.4, 0.0]]))
    assert r["hit"][0] == 1 and r["flags"][0] & oracle.FLAG_T and r["t"][0] == 1.0
    # lies in the plane z = 0 inside the bottom face: parallel (det == 0, no hit)
    r = oracle.run(Vc, Tc, np.float32([[0.2, 0.3, 0.0]]), np.float32([[0.7, 0.35, 0.0]]))
    assert r["flags"][0] & oracle.FLAG_P and r["hit"][0] == 0
    # two parallel sheets 5e-6 apart along a unit-length segment: gap in (0.1 tau, 10 tau]
    Vd = np.float32([[0, 0, 0.5], [1, 0, 0.5], [0, 1, 0.5], [0, 0, 0.505], [1, 0, 0.505], [0, 1, 0.505]])
    Td = np.int32([[0, 1, 2], [3, 4, 5]])
    r = oracle.run(Vd, Td, np.float32([[0.2, 0.2, 0.0]]), np.float32([[0.2, 0.2, 1000.0]]),)
    assert r["flags"][0] & oracle.FLAG_D
    assert r["count"][0] == 2  # gap 5e-6 > tau = 1e-6


def test_degenerate_inputs_and_validation():
    V, T = synth.fixture()
    # zero-length segment on the surface: det == 0 -> no hit
    p = np.float32([[12.5, 2.2, 1.06]])
    r = oracle.run(V, T, p, p)
    assert r["hit"][0] == 0
    # degenerate (collinear) triangle never hits
    Vd = np.float32([[0, 0, 0], [1, 1, 1], [2, 2, 2]])
    r = oracle.run(Vd, np.int32([[0, 1, 2]]), np.float32([[1, 1, 0]]), np.float32([[1, 1, 2]]))
    assert r["hit"][0] == 0
    # reading R12: a segment with a NaN / Inf coordinate is a miss
    S = np.float32([[12.5, 2.2, np.nan], [np.inf, 2.2, 2.0], [12.7, 2.2, 2.0]])
    E = np.float32([[12.5, 2.2, 0.0], [12.7, 2.2, 0.0], [12.7, 2.2, -np.inf]])
    r = oracle.run(V, T, S, E)
    assert r["hit"].tolist() == [0, 0, 0] and r["count"].tolist() == [0, 0, 0]
    with pytest.raises(ValueError):
        oracle.run(V, np.int32([[0, 1, 5]]), p, p)
    with pytest.raises(TypeError):
        oracle.run(V, T.astype(np.int64), p, p)


def test_single_pair_entry_point_matches_run():
    """rsi_oracle_mt (used by the adversarial test) agrees with rsi_oracle_run."""
    V, T = synth.fixture()
    S, E = synth.fixture_rays()
    r = oracle.run(V, T, S, E)
    for i in range(8):
        hs = [oracle.mt(S[i], E[i], *V[T[j]]) for j in range(4)]
        assert int(any(h[0] for h in hs)) == r["hit"][i]
    # exact-rational referee agrees on the paper example too
    for i in range(8):
        ts = [seg_tri_exact(S[i], E[i], *V[T[j]]) for j in range(4)]
        assert int(any(t is not None for t in ts)) == r["hit"][i]
    assert seg_tri_exact((0, 0, -1), (0, 0, 1), (-1, -1, 0), (1, -1, 0), (0, 1, 0)) == Fr(1, 2)
