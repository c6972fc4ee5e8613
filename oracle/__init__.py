"""CPU oracle for segment x triangle-mesh intersection -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product path
(``paper_2305_01867_b200``) never imports it, and it never imports the product
path.  See ``oracle/rsi_oracle.c`` for the definition it implements and the
PAPER.md passages it follows (exhaustive double-precision Moller-Trumbore,
P:13 and P:501; modes P:24-29).

Pins: ``tests/test_oracle.py`` (Fig. 3 worked example P:194-200/P:351,
exact-rational plane-clip referee, closed-form unit cube, closed-mesh parity,
canopy layer counts).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "rsi_oracle.c")
_LIB = os.path.join(_HERE, "librsi_oracle.so")
_lock = threading.Lock()
_lib = None

FLAG_E, FLAG_T, FLAG_P, FLAG_B, FLAG_D = 1, 2, 4, 8, 16
FLAG_NAMES = {FLAG_E: "edge", FLAG_T: "touch", FLAG_P: "parallel", FLAG_B: "tie", FLAG_D: "dedup"}

DEFAULT_TAU = 1e-6    # dedup tolerance in t units (reading R4)
DEFAULT_DELTA = 1e-6  # flag band (north_star "within 1e-6 (relative)")


def build(force: bool = False) -> str:
    """Compile the oracle with gcc: -O2 -ffp-contract=off, no fast-math, OpenMP."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-shared", "-fPIC", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            p = ctypes.c_void_p
            i64 = ctypes.c_int64
            lib.rsi_oracle_run.argtypes = [p, i64, p, i64, p, p, i64, ctypes.c_double,
                                           ctypes.c_double, ctypes.c_int] + [p] * 8
            lib.rsi_oracle_run.restype = ctypes.c_int
            lib.rsi_oracle_mt.argtypes = [p] * 6
            lib.rsi_oracle_mt.restype = ctypes.c_int
            lib.rsi_oracle_max_threads.restype = ctypes.c_int
            _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def max_threads() -> int:
    return int(_load().rsi_oracle_max_threads())


def mt(O, E, A, B, C):
    """One Moller-Trumbore pair in double: returns (hit, t, u, v, det)."""
    lib = _load()
    arrs = [np.ascontiguousarray(np.asarray(x, dtype=np.float64).reshape(3)) for x in (O, E, A, B, C)]
    out = np.zeros(4, np.float64)
    h = lib.rsi_oracle_mt(*[_ptr(a) for a in arrs], _ptr(out))
    return bool(h), float(out[0]), float(out[1]), float(out[2]), float(out[3])


def run(vertices, triangles, start, end, tau: float = DEFAULT_TAU,
        delta: float = DEFAULT_DELTA, threads: int = 0, flags: bool = True) -> dict:
    """Exhaustive oracle over all (ray, triangle) pairs; all three modes.

    Arguments are float32 [N_v,3] vertices, int32 [N_t,3] triangles and float32
    [N_r,3] segment start/end points.  Returns a dict of numpy
    arrays: hit (u8), count (i32), tri (i32, -1 = miss), t / dist (f64),
    point (f64 [N_r,3]), flags (u8 bitmask, if requested), nhits_raw (i32).
    """
    lib = _load()
    V = np.ascontiguousarray(vertices, dtype=np.float32).reshape(-1, 3)
    T = np.asarray(triangles)
    if T.dtype != np.int32:
        raise TypeError("triangles must be int32 (the P:272-299 int width lesson)")
    T = np.ascontiguousarray(T).reshape(-1, 3)
    S = np.ascontiguousarray(start, dtype=np.float32).reshape(-1, 3)
    E = np.ascontiguousarray(end, dtype=np.float32).reshape(-1, 3)
    if S.shape != E.shape:
        raise ValueError("start/end shape mismatch")
    nr = S.shape[0]
    out = {
        "hit": np.zeros(nr, np.uint8),
        "count": np.zeros(nr, np.int32),
        "tri": np.zeros(nr, np.int32),
        "t": np.zeros(nr, np.float64),
        "dist": np.zeros(nr, np.float64),
        "point": np.zeros((nr, 3), np.float64),
        "nhits_raw": np.zeros(nr, np.int32),
    }
    fl = np.zeros(nr, np.uint8) if flags else None
    rc = lib.rsi_oracle_run(_ptr(V), V.shape[0], _ptr(T), T.shape[0], _ptr(S), _ptr(E), nr,
                            float(tau), float(delta), int(threads),
                            _ptr(out["hit"]), _ptr(out["count"]), _ptr(out["tri"]),
                            _ptr(out["t"]), _ptr(out["dist"]), _ptr(out["point"]),
                            _ptr(fl) if fl is not None else None, _ptr(out["nhits_raw"]))
    if rc != 0:
        raise ValueError("triangle index out of range [0, N_v)")
    if fl is not None:
        out["flags"] = fl
    return out


def sparse_barycentric(res: dict):
    """The paper's barycentric return shape: (intersecting_rays,
    distances, hit_triangles, hit_points), rays ascending."""
    ids = np.nonzero(res["tri"] >= 0)[0].astype(np.int32)
    return ids, res["dist"][ids], res["tri"][ids], res["point"][ids]
