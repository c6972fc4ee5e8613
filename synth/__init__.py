"""Seeded synthetic inputs shared by tests, smoke() and bench.py.

This module holds NO intersection arithmetic: it only builds meshes (vertex /
index tables) and samples segment endpoints.  Both the CPU oracle and the CUDA
path consume its outputs; neither is imported here.

Workload shapes follow the paper (N_t ~ 1e4, N_r in [1e6, 1e8]; P:147-148:
"10M rays and a surface with 14874 vertices, 29260 triangles"; Fig. 3)
and SURVEY.md 8(d) (configs C1..C5).  Recipes are restated in DESIGN.md
"Input recipe".  All vertices/endpoints are float32, indices int32 (the
int32-everywhere lesson of P:272-299).
"""
from __future__ import annotations

import math

import numpy as np

__all__ = [
    "cube", "fixture", "fixture_rays", "canopy", "uv_sphere", "folded_terrain",
    "paper_terrain", "box_rays", "vertical_rays", "workload",
]


def _f32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


def _i32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


# --------------------------------------------------------------------------- meshes

def cube():
    """Unit cube [0,1]^3: V = {0,1}^3 with index 4x+2y+z, 12 outward-wound
    triangles, 2 per face with fixed diagonals."""
    V = [(x, y, z) for x in (0, 1) for y in (0, 1) for z in (0, 1)]
    idx = lambda x, y, z: 4 * x + 2 * y + z  # noqa: E731
    # each face: 4 corners counter-clockwise seen from outside
    faces = [
        [idx(0, 0, 0), idx(0, 0, 1), idx(0, 1, 1), idx(0, 1, 0)],  # x = 0
        [idx(1, 0, 0), idx(1, 1, 0), idx(1, 1, 1), idx(1, 0, 1)],  # x = 1
        [idx(0, 0, 0), idx(1, 0, 0), idx(1, 0, 1), idx(0, 0, 1)],  # y = 0
        [idx(0, 1, 0), idx(0, 1, 1), idx(1, 1, 1), idx(1, 1, 0)],  # y = 1
        [idx(0, 0, 0), idx(0, 1, 0), idx(1, 1, 0), idx(1, 0, 0)],  # z = 0
        [idx(0, 0, 1), idx(1, 0, 1), idx(1, 1, 1), idx(0, 1, 1)],  # z = 1
    ]
    T = []
    for a, b, c, d in faces:
        T.append((a, b, c))
        T.append((a, c, d))
    return _f32(V), _i32(T)


def fixture():
    """Fig. 3 mesh, reconstructed from the leaf AABBs printed at
    P:332-346 and the four hit points at P:200:
    square [12,13]x[2,3] split by both diagonals, centre vertex (12.5,2.5,1.1).
    T0 = bottom, T1 = right, T2 = top, T3 = left."""
    V = [(12.0, 2.0, 1.0), (13.0, 2.0, 1.2), (12.0, 3.0, 1.2), (13.0, 3.0, 1.3), (12.5, 2.5, 1.1)]
    T = [(0, 1, 4), (1, 3, 4), (2, 3, 4), (0, 2, 4)]
    return _f32(V), _i32(T)


def fixture_rays():
    """8 segments R0..R7 for the Fig. 3 scene.  R1, R2, R4, R7 are vertical
    segments through the printed hit points; the four misses are ours
    (the paper does not give ray coordinates)."""
    S = [
        (11.5, 2.5, 2.0),   # R0 outside the footprint
        (12.7, 2.2, 2.0),   # R1 -> T0 at (12.7, 2.2, 1.14)
        (12.9, 2.4, 2.0),   # R2 -> T1 at (12.9, 2.4, 1.21)
        (12.3, 2.6, 2.0),   # R3 stops above the surface
        (12.6, 2.9, 2.0),   # R4 -> T2 at (12.6, 2.9, 1.23)
        (12.1, 2.1, 2.0),   # R5 horizontal, above the surface
        (13.5, 2.2, 2.0),   # R6 outside the footprint
        (12.2, 2.4, 2.0),   # R7 -> T3 at (12.2, 2.4, 1.08)
    ]
    E = [
        (11.5, 2.5, 0.0),
        (12.7, 2.2, 0.0),
        (12.9, 2.4, 0.0),
        (12.3, 2.6, 1.5),
        (12.6, 2.9, 0.0),
        (12.9, 2.9, 2.0),
        (13.5, 2.2, 0.0),
        (12.2, 2.4, 0.0),
    ]
    return _f32(S), _f32(E)


def canopy(lift: float = 0.5):
    """Fig. 3 surface plus two patches "above triangles 1 and 2":
    copies of T1 and T2 raised by `lift` in z (patch height is ours)."""
    V, T = fixture()
    V = V.astype(np.float64)
    extra_v, extra_t = [], []
    for tri in (T[1], T[2]):
        base = len(V) + len(extra_v)
        for k in tri:
            x, y, z = V[k]
            extra_v.append((x, y, z + lift))
        extra_t.append((base, base + 1, base + 2))
    return _f32(np.vstack([V, extra_v])), _i32(np.vstack([T, extra_t]))


def uv_sphere(n_lon: int = 100, n_bands: int = 51, amp: float = 0.05):
    """Closed, mildly non-convex UV sphere:
    r = 1 + amp*sin(5 theta)*cos(7 phi); N_v = 2 + (n_bands-1)*n_lon,
    N_t = 2*n_lon*(n_bands-1).  (100, 51) -> N_t = 10 000; (1000, 501) -> 1e6."""
    rings = n_bands - 1
    k = np.arange(1, n_bands, dtype=np.float64)
    theta = math.pi * k / n_bands                       # polar angle per ring
    phi = 2.0 * math.pi * np.arange(n_lon) / n_lon
    th, ph = np.meshgrid(theta, phi, indexing="ij")     # [rings, n_lon]
    r = 1.0 + amp * np.sin(5.0 * th) * np.cos(7.0 * ph)
    ring_v = np.stack([r * np.sin(th) * np.cos(ph), r * np.sin(th) * np.sin(ph), r * np.cos(th)], -1)
    V = np.vstack([[[0.0, 0.0, 1.0]], ring_v.reshape(-1, 3), [[0.0, 0.0, -1.0]]])
    north, south = 0, 1 + rings * n_lon
    vid = lambda i, m: 1 + i * n_lon + (m % n_lon)  # noqa: E731
    T = []
    for m in range(n_lon):
        T.append((north, vid(0, m), vid(0, m + 1)))
    for i in range(rings - 1):
        for m in range(n_lon):
            a, b = vid(i, m), vid(i, m + 1)
            c, d = vid(i + 1, m), vid(i + 1, m + 1)
            T.append((a, c, d))
            T.append((a, d, b))
    for m in range(n_lon):
        T.append((south, vid(rings - 1, m + 1), vid(rings - 1, m)))
    return _f32(V), _i32(T)


def _grid_triangles(nu: int, nv: int):
    """Two triangles per cell of an nu x nv vertex grid (row-major, u fastest)."""
    i, j = np.meshgrid(np.arange(nu - 1), np.arange(nv - 1), indexing="xy")
    a = (j * nu + i).ravel()
    b, c, d = a + 1, a + nu, a + nu + 1
    T = np.empty((2 * a.size, 3), np.int64)
    T[0::2] = np.stack([a, b, d], -1)
    T[1::2] = np.stack([a, d, c], -1)
    return _i32(T)


def folded_terrain(nu: int = 101, nv: int = 51, a: float = 0.32, scale: float = 1000.0,
                   offset: float = 1000.0):
    """Recumbent S-fold: X = u - a*sin(2 pi (u - 1/2)), Y = v,
    Z = 0.3u + 0.05 sin(3 pi v), scaled x1000 and offset +1000 so coordinates are
    O(1e3) like P:414-455.  Z is monotone in u, so the sheet never
    self-intersects; vertical rays over the fold cross it 3 times.
    (101, 51) -> N_v = 5151, N_t = 10 000."""
    u = np.linspace(0.0, 1.0, nu)
    v = np.linspace(0.0, 1.0, nv)
    U, W = np.meshgrid(u, v, indexing="xy")
    X = U - a * np.sin(2.0 * math.pi * (U - 0.5))
    Y = W
    Z = 0.3 * U + 0.05 * np.sin(3.0 * math.pi * W)
    V = np.stack([X, Y, Z], -1).reshape(-1, 3) * scale + offset
    return _f32(V), _grid_triangles(nu, nv)


def paper_terrain(w: int = 134, h: int = 111, spacing: float = 24.0, seed: int = 7):
    """Paper-shaped terrain: a w x h vertex grid
    (134 x 111 -> 14 874 vertices, 29 260 triangles), ~24-unit cells at
    coordinates O(1e3), z ~ 62 +- 1.5 from a few seeded sinusoids."""
    rng = np.random.default_rng(seed)
    x = 700.0 + spacing * np.arange(w)
    y = 300.0 + spacing * np.arange(h)
    X, Y = np.meshgrid(x, y, indexing="xy")
    Z = np.full_like(X, 62.0)
    for _ in range(4):
        kx, ky = rng.uniform(0.002, 0.02, 2)
        ph = rng.uniform(0, 2 * math.pi, 2)
        Z += 0.375 * np.sin(kx * X + ph[0]) * np.cos(ky * Y + ph[1])
    V = np.stack([X, Y, Z], -1).reshape(-1, 3)
    return _f32(V), _grid_triangles(w, h)


# --------------------------------------------------------------------------- rays

def box_rays(n: int, lo, hi, seed: int):
    """Both endpoints uniform in the box [lo, hi]^3."""
    rng = np.random.default_rng(seed)
    lo = np.broadcast_to(np.asarray(lo, np.float64), (3,))
    hi = np.broadcast_to(np.asarray(hi, np.float64), (3,))
    S = rng.uniform(lo, hi, size=(n, 3))
    E = rng.uniform(lo, hi, size=(n, 3))
    return _f32(S), _f32(E)


def vertical_rays(n: int, V: np.ndarray, seed: int, overshoot: float = 0.1, jitter: float = 1e-3):
    """Near-vertical segments over the mesh footprint: from
    z_max + U(0,h) down to z_min - U(0,h), with xy jitter, where h is
    `overshoot` times the z range and the jitter is relative to the xy span."""
    rng = np.random.default_rng(seed)
    V = np.asarray(V, np.float64)
    lo, hi = V.min(0), V.max(0)
    span = hi - lo
    hz = overshoot * max(span[2], 1e-6)
    xy = rng.uniform(lo[:2], hi[:2], size=(n, 2))
    dxy = rng.uniform(-1.0, 1.0, size=(n, 2)) * jitter * span[:2]
    S = np.column_stack([xy, hi[2] + rng.uniform(0, hz, n)])
    E = np.column_stack([xy + dxy, lo[2] - rng.uniform(0, hz, n)])
    return _f32(S), _f32(E)


# --------------------------------------------------------------------------- named workloads

def workload(name: str, n_rays: int | None = None, seed: int | None = None):
    """Named configurations (BASELINE.json configs).
    Returns (V, T, S, E, mode)."""
    if name == "cube":            # configs[0]
        V, T = cube()
        S, E = box_rays(n_rays or 10_000, -0.5, 1.5, 1 if seed is None else seed)
        return V, T, S, E, "all"
    if name == "sphere":          # configs[1] / [2]
        V, T = uv_sphere()
        S, E = box_rays(n_rays or 1_000_000, -1.5, 1.5, 2 if seed is None else seed)
        return V, T, S, E, "boolean"
    if name == "terrain":         # configs[3]
        V, T = folded_terrain()
        S, E = vertical_rays(n_rays or 10_000_000, V, 4 if seed is None else seed)
        return V, T, S, E, "intercept_count"
    if name == "paper_terrain":   # P:147-148 shape
        V, T = paper_terrain()
        S, E = vertical_rays(n_rays or 10_000_000, V, 6 if seed is None else seed)
        return V, T, S, E, "boolean"
    if name == "sphere1m":        # configs[4]
        V, T = uv_sphere(1000, 501)
        S, E = box_rays(n_rays or 100_000_000, -1.5, 1.5, 5 if seed is None else seed)
        return V, T, S, E, "boolean"
    raise KeyError(name)
