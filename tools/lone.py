#!/usr/bin/env python
"""Per-chunk latency of walkers at low occupancy (GPU box, tuning only).

Usage: python tools/lone.py [SIZE_MIB] [SEG_MIB...]
Chunks a Markov stream (config-2 parameters) with the segment size forced to
SEG_MIB (so n/SEG walkers run, each alone on its SM for large SEG) and prints
us per chunk per walker.  With a -DSEQCDC_CLK=1 build (SEQCDC_LIB=...), also
the walker's cycle split: ring waits, rounds and resolve cycles per chunk."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2505_21194_b200 as sc  # noqa: E402

mib = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
segs = [int(x) for x in sys.argv[2:]] or [mib, 64, 16, 4]
n = mib << 20
p = sc.SeqParams.table1(4, 1)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
synth.fill_device("markov", 1, 0, d)
cuts = torch.empty(sc.max_cuts(n, p), dtype=torch.int64, device="cuda")
nc = torch.zeros(1, dtype=torch.int64, device="cuda")
clk = getattr(sc.lib(), "seqcdc_debug_clk", None) if os.environ.get("SEQCDC_LIB") else None
for seg in segs:
    sc.set_segment_bytes(seg << 20)
    sc.chunk_into(d, p, cuts, nc)
    torch.cuda.synchronize()
    if clk is not None:
        clk(ctypes.byref((ctypes.c_ulonglong * 8)()))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sc.chunk_into(d, p, cuts, nc)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    k = int(nc.item())
    nw = max(1, n // (seg << 20)) if seg else 1
    out = {"MiB": mib, "seg_MiB": seg, "walkers": nw, "ms": round(ms, 3), "chunks": k,
           "us_per_chunk_per_walker": round(ms * 1e3 / (k / nw), 4), "GBps": round(n / ms / 1e6, 1)}
    if clk is not None:
        a = (ctypes.c_ulonglong * 8)()
        clk(ctypes.byref(a))
        out.update({"wait_cyc_per_chunk": round(a[0] / k, 1), "rounds_per_chunk": round(a[1] / a[2], 3),
                    "resolve_cyc_per_chunk": round(a[3] / a[2], 1), "resolve_calls": a[2],
                    "ring_need_cyc_per_round": round(a[4] / a[1], 1), "classify_cyc_per_round": round(a[5] / a[1], 1),
                    "decide_cyc_per_decision": round(a[6] / max(1, a[2]), 1),
                    "issue_cyc_per_chunk": round(a[7] / k, 1)})
    print(json.dumps(out), flush=True)
sc.set_segment_bytes(0)
