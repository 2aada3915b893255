"""Whole-list parity of a GPU cut list against the CPU oracle, on all host
cores, plus the method's own bytes (SURVEY.md 8(d) "algorithmic bytes").

Why independent windows are a complete check: a chunk that starts at b is a
function of bytes [b, b + max) alone (P:179 sub-minimum skip, P:189 content
skip, P:266 max cut all restart at the chunk start).  Pick window starts
s_0 = 0 < s_1 < ... among the GPU's own cuts; window j runs the oracle from
s_j for every chunk starting before s_{j+1} and must reproduce exactly the GPU
cuts in (s_j, s_{j+1}].  If every window does, the oracle's chain from 0 passes
through every s_j and equals the GPU list (induction over j); any wrong GPU cut
makes its window differ.  The windows are independent, so they run in
parallel (ctypes releases the GIL).

Touched units: the oracle records, per unit size 2^k bytes, the distinct
stream-aligned units holding a byte of a compared pair; per window the counts
add up, minus one where a window's last unit is the next window's first."""
from __future__ import annotations

import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

import oracle

SHIFTS = (5, 7, 9, 11)        # 32 B sectors, 128 B lines, 512 B, 2 KiB


def oracle_params(w) -> "oracle.Params":
    return oracle.table1(w.avg_kib, w.mode)


def check_windows(get_bytes, n: int, p: "oracle.Params", cuts: np.ndarray, window: int = 256 << 20,
                  threads: int | None = None) -> dict:
    """`get_bytes(a, b)` -> uint8 numpy array of stream bytes [a, b).  `cuts` =
    the GPU list (uint64).  Returns bit_exact, the first mismatch, touched units,
    pairs compared and the oracle time on `threads` host threads."""
    cuts = np.ascontiguousarray(cuts, dtype=np.uint64)
    threads = threads or os.cpu_count() or 1
    out = {"bit_exact": False, "ncuts": int(cuts.size), "threads": threads}
    if n == 0:
        out["bit_exact"] = cuts.size == 0
        return out
    if cuts.size == 0 or int(cuts[-1]) != n or (cuts.size > 1 and not np.all(cuts[1:] > cuts[:-1])) or cuts[0] == 0:
        out["first_mismatch"] = "list is not a strictly increasing partition ending at n"
        return out
    # window starts: 0 and the last GPU cut at or below each multiple of `window`
    marks = np.arange(window, n, window, dtype=np.uint64)
    ks = np.searchsorted(cuts, marks, side="right")          # cuts[k-1] <= mark
    starts = sorted({0} | {int(cuts[k - 1]) for k in ks.tolist() if k > 0})
    bounds = starts + [n]

    def run(j):
        s, e = bounds[j], bounds[j + 1]
        hi = min(n, e + p.max_size) if e < n else n
        buf = get_bytes(s, hi)
        got, pairs, touch = oracle.chunk_window(buf, (e - 1 - s) if e < n else hi, p, origin=s, unit_shifts=SHIFTS)
        got = got + np.uint64(s)
        k0, k1 = int(np.searchsorted(cuts, s, side="right")), int(np.searchsorted(cuts, e, side="right"))
        want = cuts[k0:k1]
        ok = got.size == want.size and bool(np.array_equal(got, want))
        bad = None
        if not ok:
            m = min(got.size, want.size)
            d = np.nonzero(got[:m] != want[:m])[0]
            i = int(d[0]) if d.size else m
            bad = {"cut_index": k0 + i, "gpu": int(want[i]) if i < want.size else None,
                   "oracle": int(got[i]) if i < got.size else None}
        return ok, bad, pairs, touch

    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        res = list(ex.map(run, range(len(starts))))
    dt = time.perf_counter() - t0
    out["bit_exact"] = all(r[0] for r in res)
    bad = [r[1] for r in res if r[1] is not None]
    if bad:
        out["first_mismatch"] = bad[0]
    out["pairs_compared"] = sum(r[2] for r in res)
    touched = {}
    for sh in SHIFTS:
        c = sum(r[3][sh][0] for r in res)
        for a, b in zip(res[:-1], res[1:]):
            la, fb = a[3][sh][2], b[3][sh][1]
            if la == fb and la != oracle.NONE_U64:
                c -= 1
        touched[sh] = c
    out["touched_bytes"] = {f"{1 << sh}B_units": touched[sh] << sh for sh in SHIFTS}
    out["touched_fraction"] = {f"{1 << sh}B_units": round((touched[sh] << sh) / n, 5) for sh in SHIFTS}
    out["oracle_s"] = round(dt, 2)
    out["windows"] = len(starts)
    return out


def time_oracle_single(get_bytes, n: int, p: "oracle.Params", cuts: np.ndarray, budget_s: float = 10.0,
                       piece: int = 1 << 30) -> dict:
    """The oracle as it stands (plain single-threaded C loop, oracle.chunk) on
    consecutive pieces of the stream, each starting at a true cut, until
    ~budget_s of CPU time: GB/s = bytes / time (a bounded sample)."""
    work, t, pos = 0, 0.0, 0
    cuts = np.ascontiguousarray(cuts, dtype=np.uint64)
    while pos < n and t < budget_s:
        end = min(n, pos + piece)
        buf = get_bytes(pos, end)
        t0 = time.perf_counter()
        got = oracle.chunk(buf, p)
        t += time.perf_counter() - t0
        work += end - pos
        if end >= n:
            pos = n
            break
        # the next piece starts at the last cut the truncated piece cannot have
        # moved (a chunk starting >= end - max may differ from the stream's)
        safe = got[(got + np.uint64(pos)) <= np.uint64(end - p.max_size)]
        if safe.size == 0:
            break
        pos = pos + int(safe[-1])
    done = pos
    return {"GBps": round(work / t / 1e9, 4), "bytes": done, "bytes_processed": work, "seconds": round(t, 2)}
