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


# ---------------------------------------------------------------- config 4: versioned backup stream
# V0 = `base` uniform bytes (seed); version v+1 = seeded random edits of version v
# until the edit lengths sum to >= frac of its size: each edit at a uniform
# position, length U[1,4096], op insert-random / delete / overwrite-random
# (uniform), non-overlapping.  The stream is V0 || V1 || ... || V_nver.
# Only byte movement and seeded draws -- none of SeqCDC's arithmetic.
def _version_edits(rng, size: int, frac: float):
    import bisect
    budget = int(frac * size)
    starts, ends, edits = [], [], []
    total = 0
    while total < budget:
        pos = int(rng.integers(0, size))
        ln = int(rng.integers(1, 4097))
        op = int(rng.integers(0, 3))          # 0 insert, 1 delete, 2 overwrite
        end = pos if op == 0 else pos + ln
        if end > size:
            continue
        i = bisect.bisect_left(starts, pos)
        # reject overlap with the neighbours (an insert is a point at pos)
        if i > 0 and ends[i - 1] > pos:
            continue
        if i < len(starts) and starts[i] < end:
            continue
        if i < len(starts) and op == 0 and starts[i] == pos:
            continue
        starts.insert(i, pos)
        ends.insert(i, end)
        edits.insert(i, (pos, ln, op))
        total += ln
    return edits


def versions_plan(seed: int, base: int, nver: int = 10, frac: float = 0.01, max_slice: int = 1 << 16):
    """-> (sizes[nver+1], plans[nver]); plan v (building version v+1) is a uint64
    array [k,4] of (sel, src_off, dst_off, len): sel 0 = version v, 1 = the
    version's random pool (uniform bytes, seed versions_pool_seed(seed, v))."""
    sizes = [base]
    plans = []
    for v in range(nver):
        rng = np.random.default_rng([seed, 4, v])
        size = sizes[-1]
        edits = _version_edits(rng, size, frac)
        sl, cur, pool = [], 0, 0
        for pos, ln, op in edits:
            if pos > cur:
                sl.append((0, cur, pos - cur))
            if op == 0:
                sl.append((1, pool, ln)); pool += ln; cur = pos
            elif op == 1:
                cur = pos + ln
            else:
                sl.append((1, pool, ln)); pool += ln; cur = pos + ln
        if cur < size:
            sl.append((0, cur, size - cur))
        rows, dst = [], 0
        for sel, so, ln in sl:                 # split long slices for the device gather
            o = 0
            while o < ln:
                k = min(max_slice, ln - o)
                rows.append((sel, so + o, dst, k))
                dst += k
                o += k
        plans.append(np.asarray(rows, dtype=np.uint64).reshape(-1, 4))
        sizes.append(dst)
    return sizes, plans


def versions_pool_seed(seed: int, v: int) -> int:
    return (seed * 1000003 + 7919 * (v + 1)) & ((1 << 63) - 1)


def _pool_len(plan) -> int:
    m = plan[:, 0] == 1
    return int((plan[m, 1] + plan[m, 3]).max()) if m.any() else 0


def versions_host(seed: int, base: int, nver: int = 10, frac: float = 0.01):
    sizes, plans = versions_plan(seed, base, nver, frac)
    out = np.empty(sum(sizes), dtype=np.uint8)
    fill_host("uniform", seed, 0, base, out[:base])
    off = [0]
    for s in sizes:
        off.append(off[-1] + s)
    for v, plan in enumerate(plans):
        prev = out[off[v]:off[v + 1]]
        pool = fill_host("uniform", versions_pool_seed(seed, v), 0, _pool_len(plan))
        dst = out[off[v + 1]:off[v + 2]]
        for sel, so, do, ln in plan.tolist():
            dst[do:do + ln] = (pool if sel else prev)[so:so + ln]
    return out, sizes


def versions_device(seed: int, base: int, nver: int = 10, frac: float = 0.01, device="cuda"):
    import torch
    sizes, plans = versions_plan(seed, base, nver, frac)
    out = torch.empty(sum(sizes), dtype=torch.uint8, device=device)
    fill_device("uniform", seed, 0, out[:base], base)
    off = [0]
    for s in sizes:
        off.append(off[-1] + s)
    lib = _load()
    lib.synth_gather_device.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_uint64, ctypes.c_void_p]
    lib.synth_gather_device.restype = ctypes.c_int
    stream = torch.cuda.current_stream(out.device).cuda_stream
    for v, plan in enumerate(plans):
        pl = _pool_len(plan)
        pool = torch.empty(max(pl, 1), dtype=torch.uint8, device=device)
        if pl:
            fill_device("uniform", versions_pool_seed(seed, v), 0, pool, pl)
        d_plan = torch.from_numpy(plan.astype(np.int64)).to(device)
        rc = lib.synth_gather_device(out[off[v + 1]:].data_ptr(), out[off[v]:].data_ptr(), pool.data_ptr(),
                                     d_plan.data_ptr(), plan.shape[0], stream)
        if rc:
            raise RuntimeError(f"synth_gather_device failed ({rc})")
        torch.cuda.current_stream(out.device).synchronize()
    return out, sizes
