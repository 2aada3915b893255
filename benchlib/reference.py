"""bench.py --impl reference: the tier's reference arm is the CPU oracle
(there is no reference code to install: /root/reference holds only the paper
text), timed as it stands -- the plain single-threaded C loop -- on the box's
host cores, on the same workload, metric, unit and config as our arm.  Each
step is a bounded sample of the stream (a prefix starting at offset 0, which
is a true chunk start) so that the whole --steps K --warmup W run ends within a
few minutes.  Under torchrun only rank 0 runs; the other ranks exit 0."""
from __future__ import annotations

import json
import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from .common import METRIC, Workload, cpu_desc


def _host_bytes(w: Workload, n: int) -> np.ndarray:
    import synth
    out = np.empty(n, dtype=np.uint8)
    piece = 32 << 20
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 1) as ex:
        list(ex.map(lambda a: synth.fill_host(w.kind, w.seed, a, min(piece, n - a), out[a:a + piece]),
                    range(0, n, piece)))
    return out


def run(args, w: Workload) -> int:
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    import oracle
    from .verify import oracle_params
    p = oracle_params(w)
    budget_s = float(os.environ.get("SEQCDC_REF_BUDGET_S", "100"))
    probe = _host_bytes(w, min(w.n, 256 << 20))
    t0 = time.perf_counter()
    oracle.chunk(probe, p)
    rate = probe.size / (time.perf_counter() - t0)                      # bytes/s, one thread
    sample = int(min(w.n, max(probe.size, rate * budget_s / (args.steps + args.warmup))))
    sample = min(w.n, (sample + (1 << 20) - 1) & ~((1 << 20) - 1))
    host = probe if sample <= probe.size else _host_bytes(w, sample)
    view = host[:sample]
    for _ in range(args.warmup):
        oracle.chunk(view, p)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        cuts = oracle.chunk(view, p)
    dt = time.perf_counter() - t0
    value = sample * args.steps / dt / 1e9
    desc = (f"first {sample} bytes of the {w.n}-byte stream per step (a prefix from offset 0; "
            f"plain single-threaded C loop)" if sample < w.n else f"whole {w.n}-byte stream per step")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": w.config(),
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": desc,
                         "cpu": cpu_desc(), "host_cores": os.cpu_count(), "ncuts_in_sample": int(cuts.size)},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "the CPU oracle (plain single-threaded C, gcc -O2) is the reference arm: no reference code exists",
    }
    print(json.dumps(line), flush=True)
    return 0
