"""-m "not gpu": the C-ABI library loads and exports every symbol include/rsi.h declares."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2305_01867_b200 import _build
    _build.build_library()
    return ctypes.CDLL(_build.LIB)


def declared_functions():
    src = open(os.path.join(ROOT, "include", "rsi.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rsi_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("rsi_build", "rsi_intersect", "rsi_test", "rsi_free", "rsi_last_error", "rsi_version",
                     "rsi_compact_hits", "rsi_rebuild", "rsi_get_stats", "rsi_bvh_download"):
        assert required in names


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_version_and_error_string_without_gpu(lib):
    lib.rsi_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.rsi_version()
    lib.rsi_last_error.restype = ctypes.c_char_p
    assert isinstance(lib.rsi_last_error(), bytes)


def test_argument_errors_need_no_gpu(lib):
    """Argument validation happens before any CUDA call."""
    lib.rsi_build.restype = ctypes.c_int
    lib.rsi_build.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                              ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]
    h = ctypes.c_void_p()
    assert lib.rsi_build(None, 0, None, 0, None, None, ctypes.byref(h)) == 2          # RSI_E_EMPTY
    assert lib.rsi_build(None, -1, None, 3, None, None, ctypes.byref(h)) == 1         # RSI_E_INVALID_ARG
    assert lib.rsi_build(None, 3, None, 1, None, None, None) == 1
    lib.rsi_free.argtypes = [ctypes.c_void_p]
    assert lib.rsi_free(None) == 0


def test_sources_compile_for_sm100a_only():
    from paper_2305_01867_b200 import _build
    assert "arch=compute_100a,code=sm_100a" in " ".join(_build.NVCC_FLAGS)
    for p in _build.SOURCES:
        s = open(p).read()
        # the product never includes, links or loads the oracle
        assert not re.search(r'#include\s*[<"][^>"]*oracle', s) and "librsi_oracle" not in s


def test_binding_rejects_int64_indices():
    import numpy as np
    import torch

    from paper_2305_01867_b200 import rsi
    with pytest.raises(TypeError):
        rsi._dev(torch.zeros((4, 3), dtype=torch.int64), torch.int32, "triangles")
    with pytest.raises(TypeError):
        rsi.rsi_test(np.zeros((3, 3), np.float32), np.zeros((1, 3), np.int64), np.zeros((1, 3), np.float32),
                     np.zeros((1, 3), np.float32))


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2305_01867_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                s = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle", s, re.M), f


def test_binding_checks_caller_outputs():
    """Caller-provided output buffers are validated before the pointer-only C-ABI sees them."""
    import numpy as np
    import torch

    from paper_2305_01867_b200 import rsi
    n = 10
    with pytest.raises(ValueError):
        rsi._check_out({"hit": torch.zeros(n - 1, dtype=torch.uint8)}, n, "boolean", "cpu")
    with pytest.raises(TypeError):
        rsi._check_out({"count": torch.zeros(n, dtype=torch.int64)}, n, "intercept_count", "cpu")
    with pytest.raises(ValueError):
        rsi._check_out({"t": torch.zeros(n)}, n, "barycentric", "cpu")  # tri missing
    with pytest.raises(ValueError):
        rsi._check_out({"tri": torch.zeros(n, dtype=torch.int32), "point": torch.zeros(n, 2)}, n, "barycentric", "cpu")
    rsi._check_out({k: v.cpu() for k, v in rsi.alloc_outputs(n, "barycentric", "cpu").items()}, n, "barycentric", "cpu")
    with pytest.raises(ValueError):  # host call with a short output array
        rsi.rsi_test(np.zeros((3, 3), np.float32), np.zeros((1, 3), np.int32), np.zeros((5, 3), np.float32),
                     np.zeros((5, 3), np.float32), {"mode": "boolean"}, out={"hit": torch.zeros(4, dtype=torch.uint8)})


def test_binding_rejects_mismatched_host_shapes():
    """rsi_test copies n*12 bytes from each ray array: start/end of different
    lengths, or arrays that are not [n, 3], are rejected before the C-ABI."""
    import numpy as np

    from paper_2305_01867_b200 import rsi
    V, T = np.zeros((3, 3), np.float32), np.zeros((1, 3), np.int32)
    S = np.zeros((5, 3), np.float32)
    with pytest.raises(ValueError):
        rsi.rsi_test(V, T, S, np.zeros((4, 3), np.float32))
    with pytest.raises(ValueError):
        rsi.rsi_test(V, T, S.reshape(-1), S.reshape(-1))          # flat arrays
    with pytest.raises(ValueError):
        rsi.rsi_test(np.zeros((2, 6), np.float32), T, S, S)       # vertices not [n, 3]
    with pytest.raises(ValueError):
        rsi.rsi_test(V, T, S, S, {"mode": "barycentric"},         # sparse tuple into dense buffers
                     out={k: v for k, v in rsi.alloc_outputs(5, "barycentric", "cpu").items()})


def test_gather_hits_export_rejects_bad_args():
    """rsi_gather_hits validates its pointers before any launch (no GPU needed)."""
    import ctypes

    from paper_2305_01867_b200 import rsi
    lib = rsi.load()
    assert lib.rsi_gather_hits(None, None, -1, None, None, None, None, None, None, None) == 1
    assert lib.rsi_gather_hits(None, None, 10, None, None, None, None, None, None, None) == 1
    assert lib.rsi_gather_hits(None, None, 0, None, ctypes.c_void_p(16), None, None, None, None, None) == 1  # dist w/o out
