#!/usr/bin/env python
"""Quick GPU check of the walkers: whole-list parity against the oracle on a
set of streams with a forced walker, plus timings.

  python tools/lane_check.py [parity|time|both] [--walker lane|warp]"""
from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2505_21194_b200 as sc  # noqa: E402
from benchlib import verify  # noqa: E402

MiB, GiB = 1 << 20, 1 << 30
DEV = torch.device("cuda", 0)


def sp(p):
    return sc.SeqParams(p.mode, p.seq_length, p.skip_trigger, p.skip_size, p.min_size, p.max_size, p.flags)


def run_case(kind, seed, n, p, G=0, steps=0):
    d = torch.empty(n, dtype=torch.uint8, device=DEV)
    if n:
        synth.fill_device(kind, seed, 0, d)
    P = sp(p)
    cuts = torch.empty(max(sc.max_cuts(n, P), 1), dtype=torch.int64, device=DEV)
    nc = torch.zeros(1, dtype=torch.int64, device=DEV)
    sc.set_segment_bytes(G)
    ws = torch.empty(max(sc.workspace_size(n, 1, P), 1), dtype=torch.uint8, device=DEV)
    sc.chunk_into(d, P, cuts, nc, workspace=ws)
    torch.cuda.synchronize()
    ms = None
    if steps:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            sc.chunk_into(d, P, cuts, nc, workspace=ws)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
    sc.set_segment_bytes(0)
    k = int(nc.item())
    got = cuts[:k].cpu().numpy().astype(np.uint64)
    host = d.cpu().numpy()
    chk = verify.check_windows(lambda a, b: host[a:b], n, p, got, window=64 * MiB)
    return chk["bit_exact"], k, ms, chk.get("first_mismatch")


def parity():
    cases = [
        ("rampmix", 5, 64 * MiB, oracle.table1(8), 0),
        ("uniform", 1, 40 * MiB + 3, oracle.table1(8), 0),
        ("markov", 2, 48 * MiB + 7, oracle.table1(4, 1), 0),
        ("zeroheavy", 3, 32 * MiB, oracle.table1(16), 0),
        ("uniform", 4, 24 * MiB, oracle.table1(16), 1 << 16),
        ("rampmix", 6, 16 * MiB + 1, oracle.table1(8), 1 << 16),
        ("markov", 7, 16 * MiB, oracle.table1(4, 1), 3 << 16),
        ("uniform", 8, 7 * MiB + 5, oracle.Params(0, 3, 20, 64, 600, 3000), 1 << 16),
        ("markov", 9, 9 * MiB, oracle.Params(1, 4, 9, 0, 300, 900), 1 << 16),
        ("rampmix", 10, 10 * MiB, oracle.Params(0, 5, 50, 256, 4096, 16384, signed=True), 1 << 16),
        ("uniform", 11, 10 * MiB, oracle.Params(0, 4, 50, 256, 4096, 16384, pairs=True), 1 << 16),
        ("uniform", 12, 0, oracle.table1(8), 0),
        ("uniform", 13, 100, oracle.table1(8), 0),
        ("uniform", 14, 5000, oracle.table1(8), 0),
        ("uniform", 15, 20000, oracle.table1(8), 0),
    ]
    ok_all = True
    for kind, seed, n, p, G in cases:
        ok, k, _, bad = run_case(kind, seed, n, p, G)
        ok_all &= ok
        print(json.dumps({"kind": kind, "n": n, "G": G, "p": str(p), "bit_exact": ok, "ncuts": k, "bad": bad}),
              flush=True)
    # degenerate / phase-locked inputs with small forced segments (overflowing extensions)
    for name, mk in [("zeros", lambda n: np.zeros(n, np.uint8)), ("inc_ramp", lambda n: (np.arange(n) % 256).astype(np.uint8)),
                     ("dec_ramp", lambda n: (255 - np.arange(n) % 256).astype(np.uint8)),
                     ("alt2", lambda n: (np.arange(n) % 2 * 7).astype(np.uint8))]:
        for G in (0, 1 << 16):
            n = 6 * MiB + 11
            b = mk(n)
            d = torch.from_numpy(b).to(DEV)
            P = sc.SeqParams.table1(8, 0)
            sc.set_segment_bytes(G)
            got = sc.chunk(d, P).cpu().numpy().astype(np.uint64)
            sc.set_segment_bytes(0)
            want = oracle.chunk(b, oracle.table1(8))
            ok = bool(np.array_equal(got, want))
            ok_all &= ok
            print(json.dumps({"kind": name, "n": n, "G": G, "bit_exact": ok, "ncuts": int(got.size)}), flush=True)
    return ok_all


def timing():
    out = []
    for kind, seed, n, avg, mode in [("rampmix", 5, 64 * GiB, 8, 0), ("rampmix", 5, 4 * GiB + 12345, 8, 0),
                                     ("markov", 2, GiB, 4, 1), ("uniform", 1, 8 * GiB, 16, 0)]:
        ok, k, ms, _ = run_case(kind, seed, n, oracle.table1(avg, mode), 0, steps=10)
        line = {"kind": kind, "n": n, "avg": avg, "walker": os.environ.get("SEQCDC_WALKER", "auto"),
                "ms": round(ms, 4), "GBps": round(n / ms / 1e6, 1), "bit_exact": ok, "ncuts": k,
                "env": {k2: v for k2, v in os.environ.items() if k2.startswith("SEQCDC_")}}
        print(json.dumps(line), flush=True)
        out.append(line)
        torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "both"
    ok = True
    if what in ("parity", "both"):
        ok = parity()
    if what in ("time", "both"):
        timing()
    sys.exit(0 if ok else 1)
