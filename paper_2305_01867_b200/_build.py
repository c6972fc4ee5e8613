"""Ahead-of-time build of librsi.so for sm_100a (nvcc; no JIT, no torch extension).

The .so is built IN-TREE (paper_2305_01867_b200/lib/) so it travels with the
repo snapshot to the GPU box.
"""
from __future__ import annotations

import glob
import hashlib
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB_DIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIB_DIR, "librsi.so")
SOURCES = sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")))
HEADERS = sorted(glob.glob(os.path.join(PKG, "csrc", "*.cuh"))) + [os.path.join(ROOT, "include", "rsi.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


HASH_FILE = LIB + ".sha256"


def source_hash() -> str:
    """Hash of every source, header and the nvcc flags: the .so is rebuilt
    whenever it differs from the hash recorded at its build (not by mtime, so a
    pushed prebuilt .so newer than the sources is never mistaken for HEAD's)."""
    h = hashlib.sha256()
    for p in SOURCES + HEADERS:
        h.update(os.path.relpath(p, ROOT).encode())
        with open(p, "rb") as f:
            h.update(f.read())
    h.update(" ".join(NVCC_FLAGS).encode())
    return h.hexdigest()


def stale() -> bool:
    if not os.path.exists(LIB) or not os.path.exists(HASH_FILE):
        return True
    with open(HASH_FILE) as f:
        return f.read().strip() != source_hash()


def build_library(force: bool = False, verbose: bool = False) -> str:
    """Compile every csrc/*.cu into lib/librsi.so with -gencode ...sm_100a."""
    if not force and not stale():
        return LIB
    os.makedirs(LIB_DIR, exist_ok=True)
    tmp = LIB + ".tmp"
    cmd = [_nvcc(), *NVCC_FLAGS, "-o", tmp, *SOURCES]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    with open(HASH_FILE, "w") as f:
        f.write(source_hash() + "\n")
    return LIB


def build_variant(name: str, defines: dict) -> str:
    """Build lib/librsi_<name>.so with extra -D defines (tuning sweeps only)."""
    out = os.path.join(LIB_DIR, f"librsi_{name}.so")
    cmd = [_nvcc(), *NVCC_FLAGS, *[f"-D{k}={v}" for k, v in defines.items()], "-o", out, *SOURCES]
    subprocess.check_call(cmd)
    return out
