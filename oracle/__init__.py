"""CPU oracle for SeqCDC boundary detection -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product path
(``paper_2505_21194_b200``) never imports it and shares no code with it.

Three independent CPU formulations of the same method (§3.1-3.4,
P:145-231; §4):

* ``chunk``        -- the literal byte-at-a-time C loop in ``seqcdc_oracle.c``
                      (ctypes).  This is THE oracle; every GPU parity test
                      compares against it.
* ``chunk_py``     -- a pure-Python twin of the same literal loop, for tiny
                      inputs (brute force).
* ``chunk_query``  -- a structurally different numpy formulation (first
                      qualifying run vs. the SkipTrigger-th opposing pair,
                      "first set bit" / "n-th set bit"), used to
                      cross-check the literal loop.

The readings adopted where the paper is ambiguous are listed in DESIGN.md
("Readings") and in the header of ``seqcdc_oracle.c``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "seqcdc_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

INCREASING = 0
DECREASING = 1


@dataclass(frozen=True)
class Params:
    """SeqCDC parameters (Table I; min/max P:378)."""

    mode: int = INCREASING          # 0 Increasing, 1 Decreasing
    seq_length: int = 5             # L, bytes in a qualifying run
    skip_trigger: int = 50          # T, opposing pairs that trigger a skip
    skip_size: int = 256            # S, bytes skipped; 0 disables skipping
    min_size: int = 4096
    max_size: int = 16384
    signed: bool = False            # compare bytes as int8 (reading c6's alternative)
    pairs: bool = False             # L counts favourable comparisons (reading c1's alternative)

    @property
    def flags(self) -> int:
        return int(self.signed) | (2 if self.pairs else 0)

    @property
    def run_bytes(self) -> int:
        """Bytes in a qualifying run: L (c1), or L+1 when L counts comparisons."""
        return self.seq_length + 1 if self.pairs else self.seq_length

    def check(self) -> None:
        if self.mode not in (0, 1):
            raise ValueError("mode must be 0 (Increasing) or 1 (Decreasing)")
        if self.seq_length < 2:
            raise ValueError("seq_length must be >= 2")
        if self.skip_trigger < 1:
            raise ValueError("skip_trigger must be >= 1")
        if self.min_size < self.seq_length:
            raise ValueError("min_size must be >= seq_length")
        if self.max_size < self.min_size:
            raise ValueError("max_size must be >= min_size")


def table1(avg_kib: int, mode: int = INCREASING) -> Params:
    """Table I with min = avg/2, max = 2*avg (BASELINE.json configs)."""
    L, T, S = {4: (5, 55, 256), 8: (5, 50, 256), 16: (5, 50, 512)}[avg_kib]
    avg = avg_kib * 1024
    return Params(mode, L, T, S, avg // 2, 2 * avg)


def build(force: bool = False) -> str:
    """Compile the C oracle with plain gcc -O2 (no SIMD intrinsics)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-shared", "-fPIC", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        u64, u32, p = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p
        lib.oracle_chunk.restype = ctypes.c_int64
        lib.oracle_chunk.argtypes = [p, u64, u32, u32, u32, u32, u64, u64, u32, p, u64, p]
        lib.oracle_next_cut.restype = u64
        lib.oracle_next_cut.argtypes = [p, u64, u64, u32, u32, u32, u32, u64, u64, u32, p]
        lib.oracle_chunk_batch.restype = ctypes.c_int64
        lib.oracle_chunk_batch.argtypes = [p, p, u32, u32, u32, u32, u32, u64, u64, u32, p, u64, p]
        lib.oracle_chunk_window.restype = ctypes.c_int64
        lib.oracle_chunk_window.argtypes = [p, u64, u64, u32, u32, u32, u32, u64, u64, u32, p, u64, p, p]
        lib.oracle_check_params.restype = ctypes.c_int
        lib.oracle_check_params.argtypes = [u32, u32, u32, u64, u64]
        _lib = lib
    return _lib


def _as_u8(data) -> np.ndarray:
    if isinstance(data, (bytes, bytearray, memoryview)):
        return np.frombuffer(bytes(data), dtype=np.uint8)
    a = np.ascontiguousarray(np.asarray(data, dtype=np.uint8))
    return a


def max_cuts(n: int, p: Params) -> int:
    return 0 if n == 0 else -(-n // p.min_size)


def chunk(data, p: Params, return_examined: bool = False):
    """Literal C oracle over one stream.  Returns uint64 exclusive cut offsets."""
    p.check()
    b = _as_u8(data)
    n = int(b.size)
    cap = max_cuts(n, p) + 1
    cuts = np.empty(cap, dtype=np.uint64)
    ex = ctypes.c_uint64(0)
    k = _load().oracle_chunk(b.ctypes.data, n, p.mode, p.seq_length, p.skip_trigger,
                             p.skip_size, p.min_size, p.max_size, p.flags, cuts.ctypes.data, cap,
                             ctypes.addressof(ex))
    if k < 0:
        raise RuntimeError(f"oracle_chunk failed ({k})")
    out = cuts[:k].copy()
    return (out, int(ex.value)) if return_examined else out


def check_params_c(p: Params) -> int:
    """The C oracle's own parameter check (0 = accepted, 1 = rejected)."""
    return int(_load().oracle_check_params(p.mode, p.seq_length, p.skip_trigger, p.min_size, p.max_size))


class _Touch(ctypes.Structure):
    _fields_ = [("nunits", ctypes.c_uint32), ("shift", ctypes.c_uint32 * 4), ("origin", ctypes.c_uint64),
                ("first", ctypes.c_uint64 * 4), ("last", ctypes.c_uint64 * 4), ("count", ctypes.c_uint64 * 4)]


NONE_U64 = (1 << 64) - 1


def chunk_window(data, last_start: int, p: Params, origin: int = 0, unit_shifts=(5, 7, 9, 11)):
    """Chunk ``data`` from offset 0 (a chunk start), stopping after the chunk
    that starts beyond ``last_start`` (C ``oracle_chunk_window``).  Measurement
    side: the compared pairs and, per unit size 2**shift, the distinct
    ``origin``-aligned units their bytes lie in (the bytes the method reads,
    SURVEY.md 8(d)).  Returns (cuts, pairs, {shift: (count, first, last)})."""
    p.check()
    b = _as_u8(data)
    n = int(b.size)
    cap = max_cuts(min(n, last_start + p.max_size), p) + 2
    cuts = np.empty(cap, dtype=np.uint64)
    ex = ctypes.c_uint64(0)
    t = _Touch()
    t.nunits = len(unit_shifts)
    for g, sh in enumerate(unit_shifts):
        t.shift[g] = sh
        t.first[g] = t.last[g] = NONE_U64
        t.count[g] = 0
    t.origin = origin
    k = _load().oracle_chunk_window(b.ctypes.data, n, last_start, p.mode, p.seq_length, p.skip_trigger,
                                    p.skip_size, p.min_size, p.max_size, p.flags, cuts.ctypes.data, cap,
                                    ctypes.addressof(ex), ctypes.addressof(t))
    if k < 0:
        raise RuntimeError(f"oracle_chunk_window failed ({k})")
    touch = {sh: (int(t.count[g]), int(t.first[g]), int(t.last[g])) for g, sh in enumerate(unit_shifts)}
    return cuts[:k].copy(), int(ex.value), touch


def next_cut(data, base: int, p: Params) -> int:
    """f(base): the single cut ending the chunk that starts at ``base``."""
    b = _as_u8(data)
    if not 0 <= base < b.size:
        raise ValueError("base out of range")
    return int(_load().oracle_next_cut(b.ctypes.data, b.size, base, p.mode, p.seq_length,
                                       p.skip_trigger, p.skip_size, p.min_size, p.max_size,
                                       p.flags, None))


def chunk_batch(data, offsets, p: Params):
    """Independent streams data[offsets[j]:offsets[j+1]]; absolute cuts + cut index."""
    p.check()
    b = _as_u8(data)
    off = np.ascontiguousarray(np.asarray(offsets, dtype=np.uint64))
    ns = off.size - 1
    cap = sum(max_cuts(int(off[j + 1] - off[j]), p) for j in range(ns)) + 1
    cuts = np.empty(cap, dtype=np.uint64)
    idx = np.empty(ns + 1, dtype=np.uint64)
    k = _load().oracle_chunk_batch(b.ctypes.data, off.ctypes.data, ns, p.mode, p.seq_length,
                                   p.skip_trigger, p.skip_size, p.min_size, p.max_size,
                                   p.flags, cuts.ctypes.data, cap, idx.ctypes.data)
    if k < 0:
        raise RuntimeError(f"oracle_chunk_batch failed ({k})")
    return cuts[:k].copy(), idx


# --------------------------------------------------------------------------
# Pure-Python twin of the literal loop (small inputs only).
# --------------------------------------------------------------------------
def chunk_py(data, p: Params) -> list:
    p.check()
    b = bytes(_as_u8(data))
    n = len(b)
    L, T, S = p.seq_length, p.skip_trigger, p.skip_size
    run_end = p.run_bytes                          # c1 (bytes) or its comparisons alternative
    cuts, base = [], 0
    while base < n:
        limit = min(base + p.max_size, n)
        i = base + p.min_size - L
        run, opp = 1, 0
        while True:
            if i + 1 >= limit:
                cut = limit
                break
            x, y = b[i], b[i + 1]
            if p.signed:                               # int8 order
                x, y = (x ^ 0x80) - 128, (y ^ 0x80) - 128
            fav = x < y if p.mode == INCREASING else x > y
            opn = x > y if p.mode == INCREASING else x < y
            if fav:
                run += 1
                if run == run_end:
                    cut = i + 2
                    break
                i += 1
            elif opn:
                run, opp = 1, opp + 1
                if opp == T:                       # P:189, reading c2
                    i, run, opp = i + 1 + S, 1, 0  # reading c3
                    continue
                i += 1
            else:
                run = 1
                i += 1
        cuts.append(cut)
        base = cut
    return cuts


# --------------------------------------------------------------------------
# Query formulation (structurally different; numpy).
#
# combine the L-1 "favourable" masks with AND; a set bit k means
# bytes k..k+L-1 are strictly monotone; the boundary is L bytes past k.
# the skip position is the n-th set bit of the opposing mask, n =
# the SkipTrigger-th opposing pair counted from the scan anchor.
# Per chunk: anchor a = base+min-L; among pairs a..limit-2 take the first run
# start k >= a (cut k+L) and the T-th opposing pair d >= a; the earlier event
# wins; a skip re-anchors at d+1+S.
# --------------------------------------------------------------------------
def chunk_query(data, p: Params) -> np.ndarray:
    p.check()
    b = _as_u8(data).view(np.int8).astype(np.int16) if p.signed else _as_u8(data).astype(np.int16)
    n = int(b.size)
    L, T, S = p.seq_length, p.skip_trigger, p.skip_size
    if n == 0:
        return np.zeros(0, dtype=np.uint64)
    diff = b[1:] - b[:-1] if n > 1 else np.zeros(0, dtype=np.int16)
    if p.mode == INCREASING:
        fav, opn = diff > 0, diff < 0
    else:
        fav, opn = diff < 0, diff > 0
    # run_start[k] = bytes k..k+Lb-1 strictly monotone  <=> fav[k..k+Lb-2] all set
    # (Lb = bytes per qualifying run: L, or L+1 when L counts comparisons)
    cs = np.concatenate([[0], np.cumsum(fav, dtype=np.int64)])
    m = p.run_bytes - 1
    npairs = fav.size
    if npairs >= m:
        ks = np.arange(0, npairs - m + 1)
        run_start = np.nonzero(cs[ks + m] - cs[ks] == m)[0]
    else:
        run_start = np.zeros(0, dtype=np.int64)
    opp_pos = np.nonzero(opn)[0]
    cuts = []
    base = 0
    while base < n:
        limit = min(base + p.max_size, n)
        a = base + p.min_size - L
        while True:
            last_pair = limit - 2                       # pairs a..last_pair are examined
            if a > last_pair:
                cut = limit
                break
            j = np.searchsorted(run_start, a)
            k = int(run_start[j]) if j < run_start.size else None
            if k is not None and k + m - 1 > last_pair:  # run must end by pair last_pair
                k = None
            q = np.searchsorted(opp_pos, a) + T - 1
            d = int(opp_pos[q]) if q < opp_pos.size else None
            if d is not None and d > last_pair:
                d = None
            if k is not None and (d is None or k + m - 1 < d):
                cut = k + m + 1
                break
            if d is not None:
                a = d + 1 + S
                continue
            cut = limit
            break
        cuts.append(cut)
        base = cut
    return np.asarray(cuts, dtype=np.uint64)


def touched_units_query(data, p: Params, unit_shifts=(5, 7, 9, 11)) -> dict:
    """Measurement cross-check written in the query form: per chunk, the pairs
    examined are the intervals [a, e] from each anchor a (then d+1+S after
    each skip) to the pair that decides it (the run's last pair, the T-th
    opposing pair, or limit-2); the units touched are those holding a byte of
    [a, e+1].  Returns {shift: distinct unit count}.  Small inputs only."""
    p.check()
    b = _as_u8(data).view(np.int8).astype(np.int16) if p.signed else _as_u8(data).astype(np.int16)
    n = int(b.size)
    L, T, S = p.seq_length, p.skip_trigger, p.skip_size
    diff = b[1:] - b[:-1] if n > 1 else np.zeros(0, dtype=np.int16)
    fav, opn = (diff > 0, diff < 0) if p.mode == INCREASING else (diff < 0, diff > 0)
    m = p.run_bytes - 1
    intervals = []
    base = 0
    while base < n:
        limit = min(base + p.max_size, n)
        a = base + p.min_size - L
        while True:
            last_pair = limit - 2
            if a > last_pair:
                cut = limit
                break
            # first pair e >= a ending a run of m favourable pairs that starts at >= a
            e_run = None
            run = 0
            e_opp = None
            cnt = 0
            for i in range(a, last_pair + 1):
                run = run + 1 if fav[i] else 0
                if run >= m:
                    e_run = i
                    break
                if opn[i]:
                    cnt += 1
                    if cnt == T:
                        e_opp = i
                        break
            if e_run is not None:
                intervals.append((a, e_run + 1))
                cut = e_run + 2
                break
            if e_opp is not None:
                intervals.append((a, e_opp + 1))
                a = e_opp + 1 + S
                continue
            intervals.append((a, last_pair + 1))
            cut = limit
            break
        base = cut
    out = {}
    for sh in unit_shifts:
        units = set()
        for lo, hi in intervals:
            units.update(range(lo >> sh, (hi >> sh) + 1))
        out[sh] = len(units)
    return out


# --------------------------------------------------------------------------
# Dedup after chunking (§2): every chunk gets a
# collision-resistant fingerprint (SHA-256), fingerprints are compared
# against those already stored, and space savings follow Eq. 1
# (P:74-76).  Plain definitions: hashlib's SHA-256 and a Python set.
# --------------------------------------------------------------------------
def chunk_starts(cuts) -> np.ndarray:
    cuts = np.asarray(cuts, dtype=np.int64)
    return np.concatenate([[0], cuts[:-1]]) if cuts.size else np.zeros(0, np.int64)


def fingerprints(data, cuts) -> np.ndarray:
    """SHA-256 digest (32 bytes) of every chunk [c_{i-1}, c_i), c_{-1} = 0."""
    import hashlib
    b = _as_u8(data)
    mv = memoryview(b)
    cuts = np.asarray(cuts, dtype=np.int64)
    out = np.empty((cuts.size, 32), dtype=np.uint8)
    for i, (s, e) in enumerate(zip(chunk_starts(cuts).tolist(), cuts.tolist())):
        out[i] = np.frombuffer(hashlib.sha256(mv[s:e]).digest(), dtype=np.uint8)
    return out


def dedup(data, cuts):
    """-> (first_occurrence[k] bool, unique_bytes): chunk i is unique iff no
    earlier chunk has the same fingerprint; unique bytes = stored
    bytes; space savings = 1 - unique/total (Eq. 1)."""
    fp = fingerprints(data, cuts)
    cuts = np.asarray(cuts, dtype=np.int64)
    sizes = cuts - chunk_starts(cuts)
    seen, first, uniq = set(), np.zeros(cuts.size, dtype=bool), 0
    for i in range(cuts.size):
        h = fp[i].tobytes()
        if h not in seen:
            seen.add(h)
            first[i] = True
            uniq += int(sizes[i])
    return first, uniq
