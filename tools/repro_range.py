#!/usr/bin/env python
"""Replay one stress case (STRESS seed + case index) as separate range calls
with a caller workspace, synchronising after each, and print the control
words of every call.  Debug aid for timing-dependent failures."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2505_21194_b200 as sc  # noqa: E402

# a case saved by the stress replay: build/<name>.npy + .json
name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
b = np.load(f"build/{name}.npy")
meta = json.load(open(f"build/{name}.json"))
n, R = meta["n"], meta["R"]
m = meta["p"]
p = oracle.Params(m[0], m[1], m[2], m[3], m[4], m[5], signed=m[6], pairs=m[7])
q = sc.SeqParams(p.mode, p.seq_length, p.skip_trigger, p.skip_size, p.min_size, p.max_size,
                 (sc.FLAG_SIGNED if p.signed else 0) | (sc.FLAG_PAIRS if p.pairs else 0))

E = 96
print(json.dumps({"n": n, "R": R, "params": repr(p)}), flush=True)
R = [x for i, x in enumerate(R) if i == 0 or x - R[i - 1] >= p.max_size or x == n]
if R[-1] != n:
    R.append(n)
for rep in range(reps):
    for r in range(len(R) - 1):
        lo, hi = R[r], R[r + 1]
        end = n if r == len(R) - 2 else min(n, hi + (E + 1) * p.max_size)
        buf = torch.from_numpy(b[lo:end]).cuda()
        cap = sc.range_max_cuts(buf.numel(), hi - lo, q)
        spec = torch.empty(cap, dtype=torch.int64, device="cuda")
        spec_n = torch.zeros(1, dtype=torch.int64, device="cuda")
        blk = torch.zeros(3 + E, dtype=torch.int64, device="cuda")
        ws = torch.zeros(sc.workspace_size(buf.numel(), 1, q), dtype=torch.uint8, device="cuda")
        sc.range_chunk_tail_into(buf, hi - lo, lo, q, spec, spec_n, 0 if r == len(R) - 2 else E, blk, workspace=ws)
        try:
            torch.cuda.synchronize()
        except Exception as e:  # noqa: BLE001
            print(json.dumps({"rep": rep, "rank": r, "error": str(e)[:80]}), flush=True)
            sys.exit(1)
        ctrl = ws[256:256 + 64].view(torch.int32).cpu().tolist()
        print(json.dumps({"rep": rep, "rank": r, "lo": lo, "hi": hi, "ncuts": int(spec_n.item()),
                          "ctrl": {"nhand": ctrl[6], "hnext": ctrl[7], "fin": ctrl[8], "ovf": ctrl[5],
                                   "done": ctrl[4]}, "lib": sc.build_info()[30:60]}), flush=True)
