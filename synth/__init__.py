"""Seeded, block-addressable synthetic byte streams (see synth.h).

Shared input generators: the product tests/bench and the CPU oracle both take
their bytes from here.  Holds none of SeqCDC's arithmetic.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = [os.path.join(_HERE, "synth.cu"), os.path.join(_HERE, "synth.h")]
_LIB = os.path.join(_HERE, "libsynth.so")

UNIFORM, MARKOV, ZEROHEAVY, RAMPMIX = 0, 1, 2, 3
KINDS = {"uniform": UNIFORM, "markov": MARKOV, "zeroheavy": ZEROHEAVY, "rampmix": RAMPMIX}


def build(force: bool = False) -> str:
    stale = not os.path.exists(_LIB) or any(os.path.getmtime(_LIB) < os.path.getmtime(s) for s in _SRC)
    if force or stale:
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
                               "-Xcompiler", "-fPIC", "-shared", "-o", tmp, _SRC[0]])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        u64, p = ctypes.c_uint64, ctypes.c_void_p
        lib.synth_fill_host.argtypes = [ctypes.c_int, u64, u64, u64, p]
        lib.synth_fill_host.restype = ctypes.c_int
        lib.synth_fill_device.argtypes = [ctypes.c_int, u64, u64, u64, p, p]
        lib.synth_fill_device.restype = ctypes.c_int
        lib.synth_batch_layout.argtypes = [u64, ctypes.c_uint32, u64, ctypes.c_double, p, p, p]
        lib.synth_batch_layout.restype = ctypes.c_int
        _lib = lib
    return _lib


def _kind(kind) -> int:
    return KINDS[kind] if isinstance(kind, str) else int(kind)


def fill_host(kind, seed: int, pos: int, length: int, out: np.ndarray | None = None) -> np.ndarray:
    """Bytes [pos, pos+length) of stream (kind, seed), generated on the host."""
    if out is None:
        out = np.empty(length, dtype=np.uint8)
    assert out.dtype == np.uint8 and out.flags.c_contiguous and out.size >= length
    rc = _load().synth_fill_host(_kind(kind), seed, pos, length, out.ctypes.data)
    if rc:
        raise RuntimeError(f"synth_fill_host failed ({rc})")
    return out[:length]


def fill_device(kind, seed: int, pos: int, tensor, length: int | None = None, stream=None) -> None:
    """Fill a CUDA uint8 tensor (contiguous) with bytes [pos, pos+len) on the device."""
    import torch
    length = tensor.numel() if length is None else length
    assert tensor.dtype == torch.uint8 and tensor.is_cuda and tensor.is_contiguous()
    s = torch.cuda.current_stream(tensor.device) if stream is None else stream
    rc = _load().synth_fill_device(_kind(kind), seed, pos, length, tensor.data_ptr(), s.cuda_stream)
    if rc:
        raise RuntimeError(f"synth_fill_device failed ({rc})")


def batch_layout(seed: int, nstreams: int, mean_size: int, jitter: float = 0.25):
    """Config-3 layout: offsets[ns+1], kinds[ns] (50/30/20 uniform/markov/zeroheavy), seeds[ns]."""
    off = np.empty(nstreams + 1, dtype=np.uint64)
    kinds = np.empty(nstreams, dtype=np.int32)
    seeds = np.empty(nstreams, dtype=np.uint64)
    _load().synth_batch_layout(seed, nstreams, mean_size, jitter, off.ctypes.data, kinds.ctypes.data,
                               seeds.ctypes.data)
    return off, kinds, seeds


def batch_host(seed: int, nstreams: int, mean_size: int, jitter: float = 0.25):
    off, kinds, seeds = batch_layout(seed, nstreams, mean_size, jitter)
    out = np.empty(int(off[-1]), dtype=np.uint8)
    for j in range(nstreams):
        a, b = int(off[j]), int(off[j + 1])
        fill_host(int(kinds[j]), int(seeds[j]), 0, b - a, out[a:b])
    return out, off


def batch_device(seed: int, nstreams: int, mean_size: int, jitter: float = 0.25, device="cuda"):
    import torch
    off, kinds, seeds = batch_layout(seed, nstreams, mean_size, jitter)
    t = torch.empty(int(off[-1]), dtype=torch.uint8, device=device)
    for j in range(nstreams):
        a, b = int(off[j]), int(off[j + 1])
        fill_device(int(kinds[j]), int(seeds[j]), 0, t[a:b], b - a)
    return t, off
