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
    """Compile every .cu to an object in parallel, then link libseqcdc.so."""
    if not (force or stale()):
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    cu = [s for s in sources() if s.endswith(".cu")]
    objs = [os.path.join(CSRC, os.path.basename(c)[:-3] + f".{os.getpid()}.o") for c in cu]
    compile_flags = [f for f in NVCC_FLAGS if f != "-shared"]

    def comp(pair):
        src, obj = pair
        cmd = ["nvcc", *compile_flags, "-c", "-o", obj, src]
        if verbose:
            print(" ".join(cmd))
        subprocess.check_call(cmd)

    try:
        with ThreadPoolExecutor(len(cu)) as ex:
            list(ex.map(comp, zip(cu, objs)))
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs])
        os.replace(tmp, LIB)
    finally:
        for o in objs:
            if os.path.exists(o):
                os.remove(o)
    return LIB
