"""In-tree build of libseqcdc.so for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libseqcdc.so")
SOURCES = [os.path.join(CSRC, f) for f in ("seqcdc.cu", "seqcdc_device.cuh", "seqcdc_range.cu", "seqcdc_dedup.cu")]
HEADER = os.path.join(ROOT, "include", "seqcdc.h")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "--extended-lambda",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-shared",
]


def sources():
    return [s for s in SOURCES if os.path.exists(s)]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in sources() + [HEADER])


def build(force: bool = False, verbose: bool = False) -> str:
    if not (force or stale()):
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    cu = [s for s in sources() if s.endswith(".cu")]
    cmd = ["nvcc", *NVCC_FLAGS, "-o", tmp, *cu]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    return LIB
