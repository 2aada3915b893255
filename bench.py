#!/usr/bin/env python
"""SeqCDC chunking benchmark (BASELINE.json metric: SeqCDC chunking GB/s at
1/2/4/8 B200; % of HBM-read roofline; cuts bit-exact).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload = BASELINE config 5, the configuration the metric is quoted on: one
64 GiB stream (50/50 uniform random bytes and +-1 ramps of length 2-600, seed
5), Increasing, SeqLength 5, SkipTrigger 50, SkipSize 256, min 4 KiB, max
16 KiB.  One step = one pass of the whole hot path over the whole stream
(stage, classify, candidates, resolve, speculative segments, seam fix-up,
compact).  N=1: the stream resident in one GPU's HBM, one
seqcdc_chunk call per step.  N>1 (torchrun, one rank per GPU): the SAME stream
sharded into N contiguous ranges (strong scaling), stitched by the seam
protocol.  Every run checks the whole cut list against the CPU oracle.

Implementation in benchlib/ (bench infrastructure, not product code).
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg5", help="cfg5 (default, the metric's config) | cfg2 | rampmix4g")
    ap.add_argument("--bytes", type=int, default=0, help="resize the workload (testing only)")
    ap.add_argument("--no-extras", action="store_true", help="skip the secondary config-2 / 4 GiB lines")
    ap.add_argument("--profile-only", action="store_true", help="timed calls only (for ncu runs)")
    ap.add_argument("--cpu-budget", type=float, default=10.0, help="seconds of single-thread oracle timing")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    from benchlib.common import WORKLOADS
    w = WORKLOADS[args.workload]
    if args.bytes:
        w = w.resized(args.bytes)
    if args.impl == "reference":
        from benchlib import reference
        return reference.run(args, w)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus > 1 or world > 1:
        from benchlib import multi
        return multi.run(args, w)
    from benchlib import single
    return single.run(args, w)


if __name__ == "__main__":
    sys.exit(main())
