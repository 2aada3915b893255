#!/usr/bin/env python
"""Quick timing sweep (GPU box): seqcdc_chunk GB/s and phase split for one
workload.  Usage: python tools/tune.py KIND SEED SIZE_MIB AVG_KIB MODE [steps]
Env knobs (SEQCDC_WALKERS_PER_SM, SEQCDC_LIB, ...) are read by the library."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2505_21194_b200 as sc  # noqa: E402

kind, seed, mib, avg, mode = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
steps = int(sys.argv[6]) if len(sys.argv) > 6 else 10
n = mib << 20
p = sc.SeqParams.table1(avg, mode)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
synth.fill_device(kind, seed, 0, d)
cuts = torch.empty(sc.max_cuts(n, p), dtype=torch.int64, device="cuda")
nc = torch.zeros(1, dtype=torch.int64, device="cuda")
ws = torch.empty(sc.workspace_size(n, 1, p), dtype=torch.uint8, device="cuda")
for _ in range(3):
    sc.chunk_into(d, p, cuts, nc, workspace=ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(steps):
    sc.chunk_into(d, p, cuts, nc, workspace=ws)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
sc.profile_enable(True)
for _ in range(steps):
    sc.chunk_into(d, p, cuts, nc, workspace=ws)
torch.cuda.synchronize()
prof, k = sc.profile_collect()
sc.profile_enable(False)
print(json.dumps({"kind": kind, "MiB": mib, "avg": avg, "mode": mode, "env": {k2: v for k2, v in os.environ.items()
                  if k2.startswith("SEQCDC")}, "GBps": round(n / ms / 1e6, 1), "ms": round(ms, 4),
                  "walk_ms": round(prof["walk"] / k, 4), "post_ms": round(prof["post"] / k, 4),
                  "walk_GBps": round(n / (prof["walk"] / k) / 1e6, 1), "ncuts": int(nc.item()),
                  "info": sc.build_info()}))
