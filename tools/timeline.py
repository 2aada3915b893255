#!/usr/bin/env python
"""Per-segment timeline of one k_walk launch (needs a -DSEQCDC_TIMELINE variant:
tools/variants.sh "tl:-DSEQCDC_TIMELINE"; SEQCDC_LIB=build/v_tl.so).
Usage: python tools/timeline.py KIND SEED SIZE_MIB AVG_KIB MODE"""
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
cap = 16384
tl = torch.zeros(4 * cap, dtype=torch.int64, device="cuda")
L = sc.lib()
L.seqcdc_debug_timeline.argtypes = [ctypes.c_void_p, ctypes.c_uint64]
for _ in range(3):
    sc.chunk_into(d, p, cuts, nc, workspace=ws)
torch.cuda.synchronize()
L.seqcdc_debug_timeline(tl.data_ptr(), cap)
sc.chunk_into(d, p, cuts, nc, workspace=ws)
torch.cuda.synchronize()
L.seqcdc_debug_timeline(None, 0)
a = tl.cpu().numpy().reshape(-1, 4)
a = a[a[:, 0] > 0]
wid = a[:, 3] >> 32
a[:, 3] &= 0xffffffff
if os.environ.get("TL_SAVE"):
    np.save(os.environ["TL_SAVE"], np.concatenate([a, wid[:, None]], axis=1))
t0 = a[:, 0].min()
st, sp, ex = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3, (a[:, 2] - t0) / 1e3
ex = np.where(a[:, 2] > 0, ex, sp)
end = ex.max()
q = lambda x: [round(float(np.percentile(x, v)), 1) for v in (0, 10, 50, 90, 99, 100)]
print(json.dumps({"kind": kind, "MiB": mib, "avg": avg, "nseg": int(len(a)), "end_us": round(float(end), 1),
                  "start_us_pct": q(st), "spec_us_pct": q(sp - st), "ext_us_pct": q(ex - sp),
                  "finish_us_pct": q(ex), "sm_busy_frac": round(float((ex - st).sum() / (end * len(np.unique(a[:, 3])) * (len(a) / len(np.unique(a[:, 3]))))), 3),
                  "info": sc.build_info()}))
