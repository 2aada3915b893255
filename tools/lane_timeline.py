#!/usr/bin/env python
"""Per-lane timeline of one k_lwalk launch (needs a -DSEQCDC_TIMELINE build:
tools/variants.sh "tl:-DSEQCDC_TIMELINE"; SEQCDC_LIB=build/v_tl.so SEQCDC_WALKER=lane).
Usage: python tools/lane_timeline.py KIND SEED SIZE_MIB AVG_KIB MODE
Prints the distribution of speculative / extension durations and chunk counts."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2505_21194_b200 as sc  # noqa: E402

kind, seed, mib, avg, mode = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
n = mib << 20
p = sc.SeqParams.table1(avg, mode)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
synth.fill_device(kind, seed, 0, d)
cuts = torch.empty(sc.max_cuts(n, p), dtype=torch.int64, device="cuda")
nc = torch.zeros(1, dtype=torch.int64, device="cuda")
ws = torch.empty(sc.workspace_size(n, 1, p), dtype=torch.uint8, device="cuda")
cap = 1 << 18
tl = torch.zeros(4 * cap, dtype=torch.int64, device="cuda")
L = sc.lib()
L.seqcdc_debug_timeline.argtypes = [ctypes.c_void_p, ctypes.c_uint64]
for _ in range(2):
    sc.chunk_into(d, p, cuts, nc, workspace=ws)
torch.cuda.synchronize()
L.seqcdc_debug_timeline(tl.data_ptr(), cap)
st4 = (ctypes.c_uint64 * 4)()
L.seqcdc_debug_lw_stats(st4, 1)
sc.chunk_into(d, p, cuts, nc, workspace=ws)
torch.cuda.synchronize()
L.seqcdc_debug_timeline(None, 0)
L.seqcdc_debug_lw_stats(st4, 0)
stats = {"warp_steps": int(st4[0]), "groups": int(st4[1]), "fills": int(st4[2]), "chunks": int(nc.item())}
a = tl.cpu().numpy().reshape(-1, 4)
a = a[a[:, 0] > 0]
t0 = a[:, 0].min()
st = (a[:, 0] - t0) / 1e3
sp = np.where(a[:, 1] > 0, (a[:, 1] - t0) / 1e3, np.nan)
en = np.where(a[:, 2] > 0, (a[:, 2] - t0) / 1e3, np.nan)
nl = (a[:, 3] >> 32).astype(np.int64)
nx = (a[:, 3] & 0xffffffff).astype(np.int64)
q = lambda x: [round(float(np.nanpercentile(x, v)), 1) for v in (0, 10, 50, 90, 99, 99.9, 100)]
print(json.dumps({"kind": kind, "MiB": mib, "avg": avg, "lanes": int(len(a)), "end_us": round(float(np.nanmax(en)), 1),
                  "pct": [0, 10, 50, 90, 99, 99.9, 100],
                  "spec_end_us": q(sp), "ext_us": q(en - sp), "finish_us": q(en),
                  "spec_cuts": q(nl), "ext_cuts": q(nx),
                  "us_per_spec_chunk": q((sp - st) / np.maximum(nl, 1)),
                  "us_per_ext_chunk": q((en - sp) / np.maximum(nx, 1)),
                  "stats": stats, "groups_per_chunk": round(stats["groups"] / max(stats["chunks"], 1), 2),
                  "fills_per_chunk": round(stats["fills"] / max(stats["chunks"], 1), 2),
                  "steps_per_warp": round(stats["warp_steps"] / max(len(a) / 32, 1), 1),
                  "info": sc.build_info()}))
