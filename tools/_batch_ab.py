# batch-path A/B on other batch shapes (tuning only): python tools/_batch_ab.py
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_2505_21194_b200 as sc
for ns, mean, avg, kindsel in [(64, 64 << 20, 4, "uniform"), (1024, 1 << 20, 4, None), (256, 64 << 20, 8, "markov"), (16, 256 << 20, 4, None)]:
    off, kinds, seeds = synth.batch_layout(7, ns, mean)
    total = int(off[-1])
    d = torch.empty(total, dtype=torch.uint8, device="cuda")
    for j in range(ns):
        a, b = int(off[j]), int(off[j + 1])
        synth.fill_device(kindsel or int(kinds[j]), int(seeds[j]), 0, d[a:b], b - a)
    doff = torch.from_numpy(off.astype(np.int64)).cuda()
    P = sc.SeqParams.table1(avg, 0)
    cuts = torch.empty(sc.max_cuts_batch(total, ns, P), dtype=torch.int64, device="cuda")
    idx = torch.empty(ns + 1, dtype=torch.int64, device="cuda")
    nc = torch.zeros(1, dtype=torch.int64, device="cuda")
    ws = torch.empty(sc.workspace_size(total, ns, P), dtype=torch.uint8, device="cuda")
    f = lambda: sc.chunk_batch_into(d, doff, P, cuts, idx, nc, total=total, workspace=ws)
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(json.dumps({"spw": os.environ.get("SEQCDC_SEGS_PER_WALKER_X100", "default"), "ns": ns, "mean_MiB": mean >> 20,
                      "avg": avg, "kind": kindsel or "mix", "GBps": round(total / ms / 1e6, 1), "ncuts": int(nc.item())}))
    del d, cuts, ws
    torch.cuda.empty_cache()
