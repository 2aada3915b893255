#!/usr/bin/env python
"""A bare chunking target for ncu captures (no oracle, no host copies):
generate one BASELINE config's stream on the device, then call the library
`--calls` times back to back.

  python tools/ncu_target.py cfg5|cfg4|cfg2|rampmix4g [--calls K] [--bytes N]

Use with  ncu -k regex:k_walk -s <warm> -c 1 ...  to capture one launch."""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2505_21194_b200 as sc  # noqa: E402

GiB = 1 << 30


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg")
    ap.add_argument("--calls", type=int, default=3)
    ap.add_argument("--bytes", type=int, default=0)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    if a.cfg == "cfg4":
        d, _ = synth.versions_device(4, 4 * GiB)
        p = sc.SeqParams.table1(16, 0)
    else:
        kind, seed, n, avg, mode = {"cfg5": ("rampmix", 5, 64 * GiB, 8, 0),
                                    "cfg2": ("markov", 2, GiB, 4, 1),
                                    "rampmix4g": ("rampmix", 5, 4 * GiB + 12345, 8, 0)}[a.cfg]
        n = a.bytes or n
        d = torch.empty(n, dtype=torch.uint8, device=dev)
        synth.fill_device(kind, seed, 0, d)
        p = sc.SeqParams.table1(avg, mode)
    n = d.numel()
    cuts = torch.empty(sc.max_cuts(n, p), dtype=torch.int64, device=dev)
    nc = torch.zeros(1, dtype=torch.int64, device=dev)
    ws = torch.empty(sc.workspace_size(n, 1, p), dtype=torch.uint8, device=dev)
    for _ in range(a.calls):
        sc.chunk_into(d, p, cuts, nc, workspace=ws)
    torch.cuda.synchronize()
    print(a.cfg, n, int(nc.item()), sc.build_info())


if __name__ == "__main__":
    main()
