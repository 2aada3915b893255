#!/usr/bin/env python
"""NEXT-3 on the GPU: Monte-Carlo search of (SeqLength, SkipTrigger, SkipSize)
for target average chunk sizes on randomized streams, min = avg/2,
max = 2*avg.  Prints one JSON line per target with the closest grid points,
the Table I row's own mean, and the sweep's batch-chunking throughput."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2505_21194_b200 import tuner  # noqa: E402

TABLE1 = {4: (5, 55, 256), 8: (5, 50, 256), 16: (5, 50, 512)}


def main():
    ns, size = 64, 16 << 20
    off = np.zeros(ns + 1, np.int64)
    off[1:] = np.cumsum([size + 3 * j for j in range(ns)])
    d = torch.empty(int(off[-1]), dtype=torch.uint8, device="cuda")
    for j in range(ns):
        synth.fill_device("uniform", 1000 + j, 0, d[off[j]:off[j + 1]], int(off[j + 1] - off[j]))
    doff = torch.from_numpy(off).cuda()
    grid = [(L, T, S) for L in (4, 5, 6) for T in (20, 30, 40, 50, 55, 60, 80) for S in (128, 256, 512, 1024)]
    for avg in (4, 8, 16):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pts = tuner.sweep(d, doff, grid, avg)
        dt = time.perf_counter() - t0
        t1 = [p for p in pts if (p.seq_length, p.skip_trigger, p.skip_size) == TABLE1[avg]][0]
        best = tuner.candidates(pts, avg * 1024, 0.05)[:5]
        print(json.dumps({
            "target_kib": avg, "stream_bytes": int(off[-1]), "grid_points": len(grid),
            "sweep_s": round(dt, 3), "sweep_GBps_incl_host": round(int(off[-1]) * len(grid) / dt / 1e9, 1),
            "table1_row": {"L_T_S": TABLE1[avg], "mean": round(t1.mean_chunk, 1), "median": t1.median_chunk,
                           "forced_frac": round(t1.forced_frac, 4)},
            "closest": [{"L_T_S": (p.seq_length, p.skip_trigger, p.skip_size), "mean": round(p.mean_chunk, 1),
                         "median": p.median_chunk, "forced_frac": round(p.forced_frac, 4)} for p in best]}),
            flush=True)


if __name__ == "__main__":
    main()
