"""Exact-rational referees used to PIN the oracle (tests only).

These deliberately use a different formulation from the oracle's
Moller-Trumbore: segment/plane clipping followed by three half-plane
(edge-side) tests, in exact rational arithmetic (``fractions.Fraction``) on the
fp32 inputs.  Semantics follow the DESIGN.md readings: closed triangle, closed
t in [0,1], a segment parallel to the plane (n . d == 0) never hits.
"""
from __future__ import annotations

from fractions import Fraction as Fr


def _v(p):
    return tuple(Fr(float(c)) for c in p)


def _sub(a, b):
    return (a[0] - b[0], a[1] - b[1], a[2] - b[2])


def _cross(a, b):
    return (a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0])


def _dot(a, b):
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]


def seg_tri_exact(O, E, A, B, C):
    """Exact hit parameter t (Fraction) of segment O->E with closed triangle ABC,
    or None.  Plane clip: n = (B-A) x (C-A); t = n.(A-O) / n.(E-O); then the
    point P = O + t (E-O) must lie on the inner side of all three edges."""
    O, E, A, B, C = map(_v, (O, E, A, B, C))
    d = _sub(E, O)
    n = _cross(_sub(B, A), _sub(C, A))
    den = _dot(n, d)
    if den == 0:
        return None
    t = _dot(n, _sub(A, O)) / den
    if t < 0 or t > 1:
        return None
    P = (O[0] + t * d[0], O[1] + t * d[1], O[2] + t * d[2])
    for v1, v2 in ((A, B), (B, C), (C, A)):
        if _dot(n, _cross(_sub(v2, v1), _sub(P, v1))) < 0:
            return None
    return t


def brute_force_exact(V, T, S, E, tau=Fr(1, 10**6)):
    """Per ray: (hit, count, nearest tri, nearest exact t) by exhaustive exact
    clipping.  count = single-linkage clusters of exact t with threshold tau."""
    out = []
    for i in range(len(S)):
        hits = []
        for j, (a, b, c) in enumerate(T):
            t = seg_tri_exact(S[i], E[i], V[a], V[b], V[c])
            if t is not None:
                hits.append((t, j))
        if not hits:
            out.append((False, 0, -1, None))
            continue
        hits.sort()
        ts = [h[0] for h in hits]
        count = 1 + sum(1 for k in range(len(ts) - 1) if ts[k + 1] - ts[k] > tau)
        out.append((True, count, hits[0][1], hits[0][0]))
    return out


def cube_clip_exact(O, E):
    """Closed-form clip of segment O->E against the closed unit cube [0,1]^3
    (slab method in exact rationals).  Returns (count, nearest_t) where count is
    the number of boundary crossings for a segment in general position:
    [O outside and the segment meets the cube] + [E outside and it meets it];
    nearest_t is the entry t if O is outside, else the exit t if E is outside."""
    O, E = _v(O), _v(E)
    d = _sub(E, O)
    lo, hi = Fr(0), Fr(1)
    for k in range(3):
        if d[k] == 0:
            if O[k] < 0 or O[k] > 1:
                return 0, None
            continue
        t0, t1 = (0 - O[k]) / d[k], (1 - O[k]) / d[k]
        if t0 > t1:
            t0, t1 = t1, t0
        lo, hi = max(lo, t0), min(hi, t1)
    if lo > hi:
        return 0, None
    inside = lambda p: all(0 <= c <= 1 for c in p)  # noqa: E731
    o_out, e_out = not inside(O), not inside(E)
    count = int(o_out) + int(e_out)
    if count == 0:
        return 0, None
    return count, (lo if o_out else hi)
