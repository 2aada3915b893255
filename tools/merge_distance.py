#!/usr/bin/env python
"""Merge distances of the speculative seams (CPU, oracle only -- analysis tool).

For every segment start lo = s * G of a stream, the speculative chain started
at lo (as if a cut were there) is followed with the oracle's f(base) until it
lands on a cut of the true chain; the number of steps is that seam's merge
distance D (the chunks an extension re-walks).  The kernel's tail is about
max D x the lone-walker time per chunk.

  python tools/merge_distance.py [kind seed MiB avg_kib mode G]   (default: config 2)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402

a = sys.argv[1:]
kind, seed = (a[0], int(a[1])) if a else ("markov", 2)
mib, avg, mode = (int(a[2]), int(a[3]), int(a[4])) if len(a) > 4 else (1024, 4, 1)
G = int(a[5]) if len(a) > 5 else 335872          # the segment length the library picks at 22 walkers/SM
n = mib << 20
b = synth.fill_host(kind, seed, 0, n)
p = oracle.table1(avg, mode)
true = oracle.chunk(b, p)
ts = set(true.tolist())
D = []
for s in range(1, -(-n // G)):
    c, k = s * G, 0
    while c not in ts and c < n:
        c = oracle.next_cut(b, c, p)
        k += 1
    D.append(k)
D = np.array(D)
print(json.dumps({"workload": f"{mib} MiB {kind} seed {seed}, Table I {avg} KiB row, mode {mode}", "G": G,
                  "seams": int(D.size), "mean": round(float(D.mean()), 2),
                  "p50_p90_p99_max": [int(np.percentile(D, q)) for q in (50, 90, 99)] + [int(D.max())],
                  "per_chunk_merge_prob": round(1.0 / (1.0 + float(D.mean())), 4)}))
