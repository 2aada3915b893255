#!/usr/bin/env python
"""NEXT-4 reports on the GPU (analogues of the paper's Fig. 10 and Fig. 12 on
synthetic data; the datasets are not available):
  * Fig. 10: chunking throughput with content-defined skipping
    (Table I SkipSize) vs without (SkipSize 0 = BASE), same min/max;
  * Fig. 12: chunk-size distribution (percentiles) per Table I row.
One JSON line per workload."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import dataclasses  # noqa: E402

import torch  # noqa: E402

import synth  # noqa: E402
import paper_2505_21194_b200 as sc  # noqa: E402


def timed(d, p, steps=10):
    n = d.numel()
    cuts = torch.empty(sc.max_cuts(n, p), dtype=torch.int64, device="cuda")
    nc = torch.zeros(1, dtype=torch.int64, device="cuda")
    ws = torch.empty(sc.workspace_size(n, 1, p), dtype=torch.uint8, device="cuda")
    for _ in range(3):
        sc.chunk_into(d, p, cuts, nc, workspace=ws)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        sc.chunk_into(d, p, cuts, nc, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    return n / ms / 1e6, cuts[: int(nc.item())]


def main():
    n = 4 << 30
    for kind, seed, mode in (("markov", 2, 1), ("uniform", 1, 0), ("zeroheavy", 3, 0), ("rampmix", 5, 0)):
        d = torch.empty(n, dtype=torch.uint8, device="cuda")
        synth.fill_device(kind, seed, 0, d)
        for avg in (4, 8, 16):
            p = sc.SeqParams.table1(avg, mode)
            seq, cuts = timed(d, p)
            base, cuts0 = timed(d, dataclasses.replace(p, skip_size=0))
            sizes = torch.diff(cuts, prepend=torch.zeros(1, dtype=cuts.dtype, device=cuts.device))[:-1].double()
            q = torch.tensor([0.1, 0.25, 0.5, 0.75, 0.9, 0.99], dtype=torch.float64, device=sizes.device)
            pct = torch.quantile(sizes, q).tolist()
            print(json.dumps({"workload": f"4 GiB {kind}", "table1_kib": avg, "mode": mode,
                              "seq_GBps": round(seq, 1), "base_noskip_GBps": round(base, 1),
                              "skip_speedup": round(seq / base, 3),
                              "chunks": int(cuts.numel()), "chunks_noskip": int(cuts0.numel()),
                              "mean_chunk": round(float(sizes.mean()), 1),
                              "cdf_p10_p25_p50_p75_p90_p99": [int(x) for x in pct],
                              "frac_at_max": round(float((sizes == p.max_size).double().mean()), 4)}), flush=True)
        del d
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
