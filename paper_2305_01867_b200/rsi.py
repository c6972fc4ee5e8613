"""Thin ctypes binding of the C-ABI in include/rsi.h (argument marshalling only).

Every step of the path runs in librsi.so's CUDA kernels; this module only turns
torch tensors into pointers, picks the current CUDA stream and allocates the
caller-owned outputs with torch.  There is no CPU fallback: if librsi.so is
missing or no CUDA device is present, calls raise.

Names follow the C entry points (rsi_build, rsi_intersect, rsi_test, ...).
The paper's user-level call `PyCudaRSI(params).test(vertices, triangles,
raysFrom, raysTo, cfg)` is `rsi_test(..., cfg={'mode': m})`.
"""
from __future__ import annotations

import ctypes
import os
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _build

MODES = {"boolean": 0, "barycentric": 1, "intercept_count": 2}
OPT_FP64_MOLLER = 1
OPT_COUNTERS = 2
OPT_DEFERRED_STATUS = 4
OPT_APETREI = 8
OPT_ROTATE = 16
OPT_PLAIN_TREE = 32

_lock = threading.Lock()
_lib = None

_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32


class RsiError(RuntimeError):
    """A non-zero rsi_status_t; .status holds the code."""

    def __init__(self, status: int, msg: str):
        super().__init__(f"rsi status {status}: {msg}")
        self.status = status


class _Options(ctypes.Structure):
    _fields_ = [("struct_size", ctypes.c_uint32), ("flags", ctypes.c_uint32), ("dedup_tau", ctypes.c_double),
                ("debug_refit_leaves", ctypes.c_int64)]


class _Integrity(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("n_internal", "half_filled", "untouched", "bad_leaf_ids", "bad_links",
                                              "bad_boxes", "unreachable_leaves")] + [("root_ok", ctypes.c_int32)]


class _Outputs(ctypes.Structure):
    _fields_ = [("hit", _p), ("count", _p), ("tri", _p), ("t", _p), ("dist", _p), ("point", _p)]


class _Stats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in ("rays", "fp64_pairs", "fp64_rays", "overflow_rays", "nonfinite_rays",
                                               "box_tests", "mt_tests", "it_search", "it_pending", "it_idle",
                                               "iterations", "leaf_lanes", "leaf_phases")]


def lib_path() -> str:
    return _build.LIB


def load():
    """Load librsi.so (raises if it was not built -- no fallback)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = os.environ.get("RSI_LIB", _build.LIB)  # variant builds for tuning sweeps
        if not os.path.exists(path):
            raise RuntimeError(f"{path} is missing: run __graft_entry__.build() "
                               "(nvcc sm_100a); there is no CPU fallback")
        lib = ctypes.CDLL(path)
        sig = {
            "rsi_version": ([], ctypes.c_char_p),
            "rsi_last_error": ([], ctypes.c_char_p),
            "rsi_launch_count": ([], ctypes.c_uint64),
            "rsi_build": ([_p, _i64, _p, _i64, _p, _p, ctypes.POINTER(_p)], ctypes.c_int),
            "rsi_rebuild": ([_p, _p, _i64, _p, _i64, _p], ctypes.c_int),
            "rsi_intersect": ([_p, _p, _p, _i64, _i32, ctypes.POINTER(_Outputs), _p], ctypes.c_int),
            "rsi_test": ([_p, _i64, _p, _i64, _p, _p, _i64, _i32, _p, ctypes.POINTER(_Outputs), _p], ctypes.c_int),
            "rsi_compact_hits": ([_p, _i64, _p, _p, _p], ctypes.c_int),
            "rsi_gather_hits": ([_p, _p, _i64, _p, _p, _p, _p, _p, _p, _p], ctypes.c_int),
            "rsi_free": ([_p], ctypes.c_int),
            "rsi_release_cache": ([], None),
            "rsi_get_stats": ([_p, ctypes.POINTER(_Stats), _p], ctypes.c_int),
            "rsi_build_status": ([_p, _p], ctypes.c_int),
            "rsi_reset_stats": ([_p, _p], ctypes.c_int),
            "rsi_bvh_info": ([_p, ctypes.POINTER(_i64), ctypes.POINTER(_i64), _p, _p], ctypes.c_int),
            "rsi_bvh_download": ([_p, _p, _p, _p, _p, _p, _p, _p], ctypes.c_int),
            "rsi_bvh_upload": ([_p, _p, _p, _p, _i64, _p], ctypes.c_int),
            "rsi_validate": ([_p, ctypes.POINTER(_Integrity), _p], ctypes.c_int),
            "rsi_bvh_root": ([_p, ctypes.POINTER(_i64), ctypes.POINTER(_i64), _p, _p], ctypes.c_int),
            "rsi_test_sparse": ([_p, _i64, _p, _i64, _p, _p, _i64, _p, _p, _p, _p, _p, ctypes.POINTER(_i64), _p],
                                ctypes.c_int),
        }
        for name, (args, res) in sig.items():
            f = getattr(lib, name)
            f.argtypes = args
            f.restype = res
        _lib = lib
        return lib


def _check(rc: int):
    if rc != 0:
        raise RsiError(rc, load().rsi_last_error().decode())


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _dev(t: torch.Tensor, dtype, name: str, cols: int | None = 3) -> torch.Tensor:
    if not isinstance(t, torch.Tensor):
        t = torch.as_tensor(np.asarray(t))
    if t.dtype != dtype:
        if dtype == torch.int32 and t.dtype in (torch.int64, torch.uint64):
            # the case-study-1 bug: never reinterpret / silently narrow indices
            raise TypeError(f"{name} must be int32, got {t.dtype} (P:272-299: int width mismatch)")
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if cols is not None and (t.dim() != 2 or t.shape[1] != cols):
        raise ValueError(f"{name} must have shape [n, {cols}], got {tuple(t.shape)}")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (use rsi_test for host arrays)")
    return t.contiguous()


def rsi_version() -> str:
    return load().rsi_version().decode()


def rsi_launch_count() -> int:
    """Kernels the library has launched in this process (host counter)."""
    return int(load().rsi_launch_count())


@dataclass
class Options:
    fp64_moller: bool = False   # P:501 USE_DOUBLE_PRECISION_MOLLER
    dedup_tau: float = 1e-6     # reading R4
    counters: bool = False      # instrumented kernels: box / MT test counts in rsi_get_stats
    debug_refit_leaves: int = 0  # FAULT INJECTION (tests): refit only the first k leaves
    deferred_status: bool = False  # rsi_build/rsi_rebuild do not wait: check rsi_build_status
    apetrei: bool = False       # NEXT-1: 63-bit Morton codes + Apetrei build
    rotate: bool = False        # local SAH tree rotations fused into the refit (NEXT-4 tree quality)
    plain_tree: bool = False    # keep the Karras topology (no treelet restructuring): the paper's Fig. 3 tree

    def _c(self) -> _Options:
        flags = ((OPT_FP64_MOLLER if self.fp64_moller else 0) | (OPT_COUNTERS if self.counters else 0)
                 | (OPT_DEFERRED_STATUS if self.deferred_status else 0) | (OPT_APETREI if self.apetrei else 0)
                 | (OPT_ROTATE if self.rotate else 0) | (OPT_PLAIN_TREE if self.plain_tree else 0))
        return _Options(ctypes.sizeof(_Options), flags, float(self.dedup_tau), int(self.debug_refit_leaves))


class Handle:
    """Owns an rsi_handle_t (the BVH on one device)."""

    def __init__(self, ptr: int, device: torch.device):
        self._ptr = ptr
        self.device = device

    @property
    def ptr(self) -> int:
        if not self._ptr:
            raise ValueError("handle already freed")
        return self._ptr

    def free(self):
        if self._ptr:
            _check(load().rsi_free(self._ptr))
            self._ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.free()


def rsi_build(vertices: torch.Tensor, triangles: torch.Tensor, options: Options | None = None,
              stream=None) -> Handle:
    """rsi_build: LBVH over the mesh (device tensors float32 [N_v,3], int32 [N_t,3])."""
    lib = load()
    V = _dev(vertices, torch.float32, "vertices")
    T = _dev(triangles, torch.int32, "triangles")
    opt = (options or Options())._c()
    h = _p()
    with torch.cuda.device(V.device):
        _check(lib.rsi_build(V.data_ptr(), V.shape[0], T.data_ptr(), T.shape[0], ctypes.byref(opt),
                             _stream(stream), ctypes.byref(h)))
    return Handle(h.value, V.device)


def rsi_rebuild(h: Handle, vertices: torch.Tensor, triangles: torch.Tensor, stream=None) -> Handle:
    V = _dev(vertices, torch.float32, "vertices")
    T = _dev(triangles, torch.int32, "triangles")
    if V.device != h.device or T.device != h.device:
        raise ValueError(f"mesh is on {V.device}/{T.device}, the handle lives on {h.device}")
    with torch.cuda.device(V.device):
        _check(load().rsi_rebuild(h.ptr, V.data_ptr(), V.shape[0], T.data_ptr(), T.shape[0], _stream(stream)))
    return h


def alloc_outputs(n: int, mode: str, device, with_t: bool = True) -> dict:
    """torch-allocated caller-owned outputs for `mode` (see rsi_outputs_t)."""
    if mode == "boolean":
        return {"hit": torch.empty(n, dtype=torch.uint8, device=device)}
    if mode == "intercept_count":
        return {"count": torch.empty(n, dtype=torch.int32, device=device)}
    if mode == "barycentric":
        out = {"tri": torch.empty(n, dtype=torch.int32, device=device),
               "dist": torch.empty(n, dtype=torch.float32, device=device),
               "point": torch.empty((n, 3), dtype=torch.float32, device=device)}
        if with_t:
            out["t"] = torch.empty(n, dtype=torch.float32, device=device)
        return out
    raise ValueError(f"mode must be one of {list(MODES)}, got {mode!r}")


_OUT_SPEC = {"hit": (torch.uint8, 1), "count": (torch.int32, 1), "tri": (torch.int32, 1),
             "t": (torch.float32, 1), "dist": (torch.float32, 1), "point": (torch.float32, 3)}
_REQUIRED = {"boolean": "hit", "intercept_count": "count", "barycentric": "tri"}


def _check_out(out: dict, n: int, mode: str, device) -> None:
    """Caller-provided outputs: the C-ABI takes bare pointers, so dtype, size,
    contiguity and device are checked here (a short buffer would be overrun)."""
    if _REQUIRED[mode] not in out or out[_REQUIRED[mode]] is None:
        raise ValueError(f"{mode} needs out[{_REQUIRED[mode]!r}]")
    for k, v in out.items():
        if v is None or k not in _OUT_SPEC:
            continue
        dtype, cols = _OUT_SPEC[k]
        if not isinstance(v, torch.Tensor) or v.dtype != dtype:
            raise TypeError(f"out[{k!r}] must be a {dtype} tensor")
        if not v.is_contiguous() or v.numel() < n * cols:
            raise ValueError(f"out[{k!r}] must be contiguous with >= {n * cols} elements")
        if torch.device(device) != v.device:
            raise ValueError(f"out[{k!r}] is on {v.device}, expected {device}")


def _outputs_struct(out: dict) -> _Outputs:
    o = _Outputs()
    for k in ("hit", "count", "tri", "t", "dist", "point"):
        if out.get(k) is not None:
            setattr(o, k, out[k].data_ptr())
    return o


def rsi_intersect(h: Handle, start: torch.Tensor, end: torch.Tensor, mode: str = "boolean",
                  out: dict | None = None, stream=None) -> dict:
    """rsi_intersect: per-ray traversal + Moller-Trumbore; returns the output dict."""
    if mode not in MODES:
        raise ValueError(f"mode must be one of {list(MODES)}, got {mode!r}")
    S = _dev(start, torch.float32, "start")
    E = _dev(end, torch.float32, "end")
    if S.shape != E.shape:
        raise ValueError("start/end shape mismatch")
    if S.device != E.device:
        raise ValueError(f"start is on {S.device}, end on {E.device}")
    if S.device != h.device:
        raise ValueError(f"rays are on {S.device}, the handle's BVH on {h.device}")
    n = S.shape[0]
    if out is None:
        out = alloc_outputs(n, mode, S.device)
    else:
        _check_out(out, n, mode, S.device)
    o = _outputs_struct(out)
    with torch.cuda.device(S.device):
        _check(load().rsi_intersect(h.ptr, S.data_ptr(), E.data_ptr(), n, MODES[mode], ctypes.byref(o),
                                    _stream(stream)))
    return out


def rsi_compact_hits(tri: torch.Tensor, stream=None):
    """Step 3a: ascending ray ids with tri >= 0, on the device.
    Returns (ids_buffer [n] int32, n_hits int32 device scalar)."""
    T = _dev(tri, torch.int32, "tri", cols=None)
    ids = torch.empty(T.numel(), dtype=torch.int32, device=T.device)
    nh = torch.empty(1, dtype=torch.int32, device=T.device)
    with torch.cuda.device(T.device):
        _check(load().rsi_compact_hits(T.data_ptr(), T.numel(), ids.data_ptr(), nh.data_ptr(), _stream(stream)))
    return ids, nh


def rsi_gather_hits(ids: torch.Tensor, n_hits: torch.Tensor, out: dict, stream=None) -> dict:
    """The values of the compacted hit rays (rsi_gather_hits), on the
    device: tri / dist / point rows of the ids rsi_compact_hits wrote (the hit
    count stays on the device).  Returns capacity-n buffers."""
    tri = _dev(out["tri"], torch.int32, "tri", cols=None)
    n = tri.numel()
    dist, point = out.get("dist"), out.get("point")
    g = {"tri": torch.empty(n, dtype=torch.int32, device=tri.device),
         "dist": torch.empty(n, dtype=torch.float32, device=tri.device) if dist is not None else None,
         "point": torch.empty((n, 3), dtype=torch.float32, device=tri.device) if point is not None else None}
    if dist is not None:
        _check_out({"tri": tri, "dist": dist}, n, "barycentric", tri.device)
    if point is not None:
        _check_out({"tri": tri, "point": point}, n, "barycentric", tri.device)
    ptr = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
    with torch.cuda.device(tri.device):
        _check(load().rsi_gather_hits(ids.data_ptr(), n_hits.data_ptr(), n, tri.data_ptr(), ptr(dist), ptr(point),
                                      g["tri"].data_ptr(), ptr(g["dist"]), ptr(g["point"]), _stream(stream)))
    return g


def sparse_barycentric(out: dict, stream=None):
    """The paper's barycentric return: (intersecting_rays, distances,
    hit_triangles, hit_points), rays ascending.  Compaction (3a) and the gather
    of the hit rows run in the library's kernels; the host reads the hit count
    to trim the views."""
    ids, nh = rsi_compact_hits(out["tri"], stream)
    g = rsi_gather_hits(ids, nh, out, stream)
    k = int(nh.item())
    return ids[:k], g["dist"][:k], g["tri"][:k], g["point"][:k]


def rsi_test(vertices, triangles, start, end, cfg: dict | None = None, options: Options | None = None,
             stream=None, out: dict | None = None, sparse: bool = True):
    """End-to-end on HOST arrays through the C-ABI's rsi_test:
    H2D, build, intersect, D2H, synchronize.  Returns the boolean array, the
    counts, or (intersecting_rays, distances, hit_triangles, hit_points) -- the
    paper's sparse tuple, compacted and gathered on the device (rsi_test_sparse);
    sparse=False returns the dense output dict instead (into `out` if given).
    Every array must have shape [n, 3]; start and end must match."""
    lib = load()
    mode = (cfg or {}).get("mode", "boolean")
    if mode not in MODES:
        raise ValueError(f"mode must be one of {list(MODES)}, got {mode!r}")

    def host(a, dtype, name):
        if isinstance(a, torch.Tensor):
            if a.is_cuda:
                raise ValueError(f"{name}: rsi_test takes host arrays")
            if a.dtype != dtype:
                raise TypeError(f"{name} must be {dtype}, got {a.dtype}")
            t = a.contiguous()
        else:
            a = np.asarray(a)
            nd = {torch.float32: np.float32, torch.int32: np.int32}[dtype]
            if a.dtype != nd:
                raise TypeError(f"{name} must be {nd.__name__}, got {a.dtype} (P:272-299)")
            t = torch.from_numpy(np.ascontiguousarray(a))
        # the C-ABI reads n * 12 bytes per array: the shape must be exactly [n, 3]
        if t.dim() != 2 or t.shape[1] != 3:
            raise ValueError(f"{name} must have shape [n, 3], got {tuple(t.shape)}")
        return t

    V = host(vertices, torch.float32, "vertices")
    T = host(triangles, torch.int32, "triangles")
    S = host(start, torch.float32, "start")
    E = host(end, torch.float32, "end")
    if S.shape != E.shape:
        raise ValueError(f"start {tuple(S.shape)} and end {tuple(E.shape)} differ in shape")
    n = S.shape[0]
    opt = (options or Options())._c()
    if mode == "barycentric" and sparse and out is not None:
        # the sparse tuple is compacted on the device (rsi_test_sparse, step 3a);
        # caller-provided buffers receive the DENSE per-ray outputs
        raise ValueError("out= receives the dense per-ray outputs: pass sparse=False "
                         "(or omit out for the sparse tuple, compacted on the device)")
    if mode == "barycentric" and sparse:
        # the paper's sparse tuple: compaction and gather on the device
        ids = np.empty(n, np.int32)
        dist = np.empty(n, np.float32)
        tri = np.empty(n, np.int32)
        point = np.empty((n, 3), np.float32)
        nh = _i64()
        ptr = lambda a: a.ctypes.data_as(_p)  # noqa: E731
        _check(lib.rsi_test_sparse(V.data_ptr(), V.shape[0], T.data_ptr(), T.shape[0], S.data_ptr(), E.data_ptr(), n,
                                   ctypes.byref(opt), ptr(ids), ptr(dist), ptr(tri), ptr(point), ctypes.byref(nh),
                                   _stream(stream)))
        m = nh.value
        return ids[:m], dist[:m], tri[:m], point[:m]
    if out is None:
        out = {k: v.cpu() for k, v in alloc_outputs(n, mode, "cpu").items()}
    else:
        _check_out(out, n, mode, "cpu")
    o = _outputs_struct(out)
    _check(lib.rsi_test(V.data_ptr(), V.shape[0], T.data_ptr(), T.shape[0], S.data_ptr(), E.data_ptr(), n,
                        MODES[mode], ctypes.byref(opt), ctypes.byref(o), _stream(stream)))
    if mode == "boolean":
        return out["hit"].numpy().view(np.bool_).reshape(n, 1)  # 0/1 bytes: a view, no copy
    if mode == "intercept_count":
        return out["count"].numpy()
    return out  # barycentric, sparse=False: the dense per-ray outputs


def rsi_build_status(h: Handle, stream=None):
    """Raise the device-side input-check error of the last (deferred) build, if any."""
    _check(load().rsi_build_status(h.ptr, _stream(stream)))


def rsi_get_stats(h: Handle, stream=None) -> dict:
    st = _Stats()
    _check(load().rsi_get_stats(h.ptr, ctypes.byref(st), _stream(stream)))
    return {n: int(getattr(st, n)) for n, _ in _Stats._fields_}


def rsi_reset_stats(h: Handle, stream=None):
    _check(load().rsi_reset_stats(h.ptr, _stream(stream)))


def rsi_free(h: Handle):
    h.free()


def rsi_release_cache():
    """Free this thread's cached rsi_test workspace."""
    load().rsi_release_cache()


def rsi_bvh_info(h: Handle) -> dict:
    nt, nn = _i64(), _i64()
    lo = (ctypes.c_float * 3)()
    hi = (ctypes.c_float * 3)()
    _check(load().rsi_bvh_info(h.ptr, ctypes.byref(nt), ctypes.byref(nn), lo, hi))
    return {"n_triangles": nt.value, "n_nodes": nn.value, "scene_lo": list(lo), "scene_hi": list(hi)}


def rsi_bvh_download(h: Handle, stream=None) -> dict:
    """Copy the BVH to host numpy arrays (P:204-241 debugging strategy)."""
    info = rsi_bvh_info(h)
    nt, nn = info["n_triangles"], info["n_nodes"]
    d = {
        "child": np.zeros((nn, 2), np.int32),
        "box": np.zeros((nn, 2, 6), np.float32),
        "leaf_tri": np.zeros(nt, np.int32),
        "morton": np.zeros(nt, np.uint32),
        "parent": np.zeros(nn + nt, np.int32),
        "arrivals": np.zeros(nn, np.uint32),
    }
    ptrs = [d[k].ctypes.data_as(_p) for k in ("child", "box", "leaf_tri", "morton", "parent", "arrivals")]
    _check(load().rsi_bvh_download(h.ptr, *ptrs, _stream(stream)))
    d.update(info)
    d.update(rsi_bvh_root(h, stream))
    return d


def rsi_bvh_upload(h: Handle, child, box, leaf_tri, root: int, stream=None) -> None:
    """Replace the handle's binary tree by a host-given one over the same mesh
    (the layout of rsi_bvh_download: child [n_nodes, 2] int32, box [n_nodes, 2, 6]
    float32, leaf_tri [N_t] int32, root node) and rebuild the 4-wide records."""
    info = rsi_bvh_info(h)
    nt, nn = info["n_triangles"], info["n_nodes"]
    child = np.ascontiguousarray(child, np.int32)
    box = np.ascontiguousarray(box, np.float32)
    leaf_tri = np.ascontiguousarray(leaf_tri, np.int32)
    if child.shape != (nn, 2) or box.shape != (nn, 2, 6) or leaf_tri.shape != (nt,):
        raise ValueError(f"upload shapes {child.shape} {box.shape} {leaf_tri.shape} for N_t={nt}, n_nodes={nn}")
    _check(load().rsi_bvh_upload(h.ptr, child.ctypes.data_as(_p), box.ctypes.data_as(_p),
                                 leaf_tri.ctypes.data_as(_p), int(root), _stream(stream)))


def rsi_bvh_root(h: Handle, stream=None) -> dict:
    """Root node, sentinel (-1 unless RSI_OPT_APETREI) and the sorted full-width codes."""
    root, sent = _i64(), _i64()
    n = rsi_bvh_info(h)["n_triangles"]
    m63 = np.zeros(n, np.uint64)
    _check(load().rsi_bvh_root(h.ptr, ctypes.byref(root), ctypes.byref(sent), m63.ctypes.data_as(_p), _stream(stream)))
    return {"root": root.value, "sentinel": sent.value, "morton63": m63}


def rsi_validate(h: Handle, stream=None) -> dict:
    """GPU integrity check.  Returns the report dict with
    "ok" = True for a valid tree (RSI_E_INTEGRITY is reported, not raised)."""
    rep = _Integrity()
    rc = load().rsi_validate(h.ptr, ctypes.byref(rep), _stream(stream))
    if rc not in (0, 7):
        _check(rc)
    d = {n: int(getattr(rep, n)) for n, _ in _Integrity._fields_}
    d["ok"] = rc == 0
    return d


class PyCudaRSI:
    """The paper's user-facing call shape:

        with PyCudaRSI(design_params) as pycu:
            ray_intersects = pycu.test(vertices, triangles, raysFrom, raysTo, {'mode': 'boolean'})
            (intersecting_rays, distances, hit_triangles, hit_points) = pycu.test(..., {'mode': 'barycentric'})

    design_params: 'USE_DOUBLE_PRECISION_MOLLER' -> every Moller-Trumbore
    test in double (results are identical either way);
    'USE_EXTRA_BVH_FIELDS' (a debugging layout of the paper's node
    struct) is accepted and has no effect -- the tree is inspected through
    rsi_bvh_download / diagnostics instead.  Thin wrapper over rsi_test /
    rsi_test_sparse; leaving the context releases the cached device workspace."""

    _KNOWN = {"USE_DOUBLE_PRECISION_MOLLER", "USE_EXTRA_BVH_FIELDS"}

    def __init__(self, design_params: dict | None = None):
        params = dict(design_params or {})
        unknown = set(params) - self._KNOWN
        if unknown:
            raise ValueError(f"unknown design_params {sorted(unknown)}; known: {sorted(self._KNOWN)}")
        self.options = Options(fp64_moller=bool(params.get("USE_DOUBLE_PRECISION_MOLLER", False)))

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        rsi_release_cache()

    def test(self, vertices, triangles, raysFrom, raysTo, cfg: dict | None = None):
        return rsi_test(vertices, triangles, raysFrom, raysTo, cfg, self.options)
