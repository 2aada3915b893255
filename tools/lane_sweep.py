#!/usr/bin/env python
"""Sweep lane-walker knobs (environment, read per call) on one resident stream.

  python tools/lane_sweep.py [cfg5|rampmix16g] 'ENV=V,ENV2=W' ...

Prints one JSON line per setting: ms per call (CUDA events, 5 calls after one
warm-up), the cut count (must not change), and the per-kernel split from the
library's profile hooks."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2505_21194_b200 as sc  # noqa: E402

GiB = 1 << 30
which = sys.argv[1]
n = {"cfg5": 64 * GiB, "rampmix8g": 8 * GiB, "rampmix12g": 12 * GiB, "rampmix16g": 16 * GiB, "rampmix32g": 32 * GiB}[which]
d = torch.empty(n, dtype=torch.uint8, device="cuda")
synth.fill_device("rampmix", 5, 0, d)
p = sc.SeqParams.table1(8, 0)
cuts = torch.empty(sc.max_cuts(n, p), dtype=torch.int64, device="cuda")
nc = torch.zeros(1, dtype=torch.int64, device="cuda")
for spec in sys.argv[2:] or [""]:
    env = dict(kv.split("=") for kv in spec.split(",") if kv)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    ws = torch.empty(sc.workspace_size(n, 1, p), dtype=torch.uint8, device="cuda")
    sc.chunk_into(d, p, cuts, nc, workspace=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        sc.chunk_into(d, p, cuts, nc, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    sc.profile_enable(True)
    for _ in range(3):
        sc.chunk_into(d, p, cuts, nc, workspace=ws)
    torch.cuda.synchronize()
    prof, k = sc.profile_collect()
    sc.profile_enable(False)
    print(json.dumps({"stream": which, "env": env, "ms": round(ms, 4), "GBps": round(n / ms / 1e6, 1),
                      "ncuts": int(nc.item()), "walk_ms": round(prof["walk"] / k, 4),
                      "post_ms": round(prof["post"] / k, 4), "lib": sc.build_info()[:80]}), flush=True)
    del ws
    for k2, v in old.items():
        if v is None:
            os.environ.pop(k2, None)
        else:
            os.environ[k2] = v
