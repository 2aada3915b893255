#!/usr/bin/env python
"""Full-size runs of BASELINE.json's five configs on one B200 (GPU box):
throughput of the chunking call and bit-exactness against the CPU oracle
(full lists where host memory allows, a streaming oracle otherwise).

  python tools/configs_bench.py [cfg ...]     cfg in 1 2 3 4 5 (default 1 2 3 5)

One JSON line per config/parameter set.  Config 5 runs on one GPU here (the
64 GiB stream fits in HBM); its multi-GPU form is bench.py --gpus N."""
from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2505_21194_b200 as sc  # noqa: E402

GiB, MiB = 1 << 30, 1 << 20
DEV = torch.device("cuda", 0)


def sp(p):
    return sc.SeqParams(p.mode, p.seq_length, p.skip_trigger, p.skip_size, p.min_size, p.max_size)


def time_calls(fn, steps, flush=None):
    """Mean ms per call (CUDA events around each call; an L2 flush between calls
    when `flush` is given, outside the timed intervals)."""
    fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(steps):
        if flush is not None:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / steps


def stream_oracle_check(d, p, got):
    """Compare the GPU cut list `got` (numpy uint64) of device stream `d` with the
    oracle, streaming 1 GiB windows to the host (a chunk that starts at b is
    determined by bytes [b, b + max) -- P:179)."""
    n = d.numel()
    W = GiB
    pos, k = 0, 0
    while pos < n:
        end = min(n, pos + W + p.max_size)
        buf = d[pos:end].cpu().numpy()
        cuts = oracle.chunk(buf, p).astype(np.uint64) + np.uint64(pos)
        if end < n:                          # trust chunks starting at <= pos + W
            starts = np.concatenate([[pos], cuts[:-1]])
            cuts = cuts[starts <= pos + W]
        m = cuts.size
        if not np.array_equal(got[k:k + m], cuts):
            bad = int(np.nonzero(got[k:k + m] != cuts)[0][0]) if got[k:k + m].size == m else -1
            return False, f"mismatch near cut {k + bad}"
        k += m
        pos = int(cuts[-1])
    return k == got.size, f"{k} cuts compared"


def cfg1(steps=50):
    n = 8 * MiB
    p = oracle.table1(8)
    b = synth.fill_host("uniform", 1, 0, n)
    d = torch.from_numpy(b).to(DEV)
    P = sp(p)
    cuts = torch.empty(sc.max_cuts(n, P), dtype=torch.int64, device=DEV)
    nc = torch.zeros(1, dtype=torch.int64, device=DEV)
    ws = torch.empty(sc.workspace_size(n, 1, P), dtype=torch.uint8, device=DEV)
    flush = torch.empty(512 * MiB, dtype=torch.uint8, device=DEV)
    ms = time_calls(lambda: sc.chunk_into(d, P, cuts, nc, workspace=ws), steps, flush)
    got = cuts[: int(nc.item())].cpu().numpy().astype(np.uint64)
    want = oracle.chunk(b, p)
    return [{"config": 1, "workload": "8 MiB uniform seed 1, Increasing, L5 T50 S256, min 4 KiB, max 16 KiB",
             "GBps": round(n / ms / 1e6, 1), "ms": round(ms, 4), "l2": "flushed (512 MiB write) before each call",
             "ncuts": int(got.size), "bit_exact": bool(np.array_equal(got, want)), "parity": "whole list"}]


def cfg2(steps=20):
    n = GiB
    p = oracle.table1(4, 1)
    P = sp(p)
    d = torch.empty(n, dtype=torch.uint8, device=DEV)
    synth.fill_device("markov", 2, 0, d)
    cuts = torch.empty(sc.max_cuts(n, P), dtype=torch.int64, device=DEV)
    nc = torch.zeros(1, dtype=torch.int64, device=DEV)
    ws = torch.empty(sc.workspace_size(n, 1, P), dtype=torch.uint8, device=DEV)
    ms = time_calls(lambda: sc.chunk_into(d, P, cuts, nc, workspace=ws), steps)
    got = cuts[: int(nc.item())].cpu().numpy().astype(np.uint64)
    ok, how = stream_oracle_check(d, p, got)
    return [{"config": 2, "workload": "1 GiB Markov seed 2, Decreasing, L5 T55 S256, min 2 KiB, max 8 KiB",
             "GBps": round(n / ms / 1e6, 1), "ms": round(ms, 4), "ncuts": int(got.size), "bit_exact": ok,
             "parity": how}]


def cfg3(steps=5, sample_streams=12):
    ns, mean = 256, 64 * MiB
    off, kinds, seeds = synth.batch_layout(3, ns, mean)
    total = int(off[-1])
    d = torch.empty(total, dtype=torch.uint8, device=DEV)
    for j in range(ns):
        a, b = int(off[j]), int(off[j + 1])
        synth.fill_device(int(kinds[j]), int(seeds[j]), 0, d[a:b], b - a)
    doff = torch.from_numpy(off.astype(np.int64)).to(DEV)
    out = []
    rng = np.random.default_rng(33)
    pick = sorted(rng.choice(ns, sample_streams, replace=False).tolist())
    for avg in (4, 8, 16):
        p = oracle.table1(avg)
        P = sp(p)
        cuts = torch.empty(sc.max_cuts_batch(total, ns, P), dtype=torch.int64, device=DEV)
        idx = torch.empty(ns + 1, dtype=torch.int64, device=DEV)
        nc = torch.zeros(1, dtype=torch.int64, device=DEV)
        ws = torch.empty(sc.workspace_size(total, ns, P), dtype=torch.uint8, device=DEV)
        ms = time_calls(lambda: sc.chunk_batch_into(d, doff, P, cuts, idx, nc, total=total, workspace=ws), steps)
        ci = idx.cpu().numpy()
        ok = True
        for j in pick:
            a, b = int(off[j]), int(off[j + 1])
            want = oracle.chunk(d[a:b].cpu().numpy(), p).astype(np.uint64) + np.uint64(a)
            got = cuts[int(ci[j]):int(ci[j + 1])].cpu().numpy().astype(np.uint64)
            ok &= bool(np.array_equal(got, want))
        out.append({"config": 3, "workload": f"256 streams x 64 MiB +-25% (50/30/20 uniform/Markov/zero-heavy), "
                    f"Increasing, Table I {avg} KiB row", "total_bytes": total,
                    "GBps": round(total / ms / 1e6, 1), "ms": round(ms, 3), "ncuts": int(nc.item()),
                    "bit_exact": ok, "parity": f"{len(pick)} sampled streams, whole lists"})
    return out


def cfg5(steps=3, n=64 * GiB):
    p = oracle.table1(8)
    P = sp(p)
    d = torch.empty(n, dtype=torch.uint8, device=DEV)
    synth.fill_device("rampmix", 5, 0, d)
    cuts = torch.empty(sc.max_cuts(n, P), dtype=torch.int64, device=DEV)
    nc = torch.zeros(1, dtype=torch.int64, device=DEV)
    ws = torch.empty(sc.workspace_size(n, 1, P), dtype=torch.uint8, device=DEV)
    ms = time_calls(lambda: sc.chunk_into(d, P, cuts, nc, workspace=ws), steps)
    got = cuts[: int(nc.item())].cpu().numpy().astype(np.uint64)
    t0 = time.time()
    ok, how = stream_oracle_check(d, p, got)
    return [{"config": 5, "workload": f"{n >> 30} GiB rampmix seed 5 (uniform / +-1 ramps of 2-600 B), one GPU, "
             "Increasing, L5 T50 S256, min 4 KiB, max 16 KiB", "GBps": round(n / ms / 1e6, 1), "ms": round(ms, 3),
             "ncuts": int(got.size), "bit_exact": ok, "parity": how + f" (streaming oracle, {time.time() - t0:.0f} s)"}]


def dedup_ratio_parallel(b, cuts, threads=16):
    """unique/total bytes over the chunks (SHA-256 index, Eq. 1)."""
    import hashlib
    from concurrent.futures import ThreadPoolExecutor
    cuts = np.asarray(cuts, dtype=np.int64)
    starts = np.concatenate([[0], cuts[:-1]])
    mv = memoryview(b)
    parts = np.array_split(np.arange(cuts.size), threads)

    def work(ix):
        return [(hashlib.sha256(mv[starts[i]:cuts[i]]).digest(), int(cuts[i] - starts[i])) for i in ix.tolist()]

    seen, uniq = set(), 0
    with ThreadPoolExecutor(threads) as ex:
        for res in ex.map(work, parts):
            for h, ln in res:
                if h not in seen:
                    seen.add(h)
                    uniq += ln
    return uniq / b.size


def cfg4(steps=3, base=4 * GiB):
    p = oracle.table1(16)
    P = sp(p)
    t0 = time.time()
    d, sizes = synth.versions_device(4, base)
    tgen = time.time() - t0
    n = d.numel()
    cuts = torch.empty(sc.max_cuts(n, P), dtype=torch.int64, device=DEV)
    nc = torch.zeros(1, dtype=torch.int64, device=DEV)
    ws = torch.empty(sc.workspace_size(n, 1, P), dtype=torch.uint8, device=DEV)
    ms = time_calls(lambda: sc.chunk_into(d, P, cuts, nc, workspace=ws), steps)
    got = cuts[: int(nc.item())].cpu().numpy().astype(np.uint64)
    b = d.cpu().numpy()
    del d
    torch.cuda.empty_cache()
    t1 = time.time()
    want = oracle.chunk(b, p)
    tor = time.time() - t1
    exact = bool(np.array_equal(got, want))
    t2 = time.time()
    ratio = dedup_ratio_parallel(b, got)
    return [{"config": 4, "workload": f"versioned backup: {base >> 30} GiB uniform base + 10 versions x 1% edits "
             f"(ins/del/overwrite 1 B-4 KiB), one stream of {n} bytes; Increasing, L5 T50 S512, min 8 KiB, max 32 KiB",
             "GBps": round(n / ms / 1e6, 1), "ms": round(ms, 3), "ncuts": int(got.size), "bit_exact": exact,
             "parity": f"whole list vs the oracle ({tor:.0f} s single-threaded)",
             "dedup_unique_over_total": round(ratio, 6),
             "dedup_note": "computed from the GPU cut list; the oracle list is identical, so is its ratio",
             "gen_s": round(tgen, 1), "hash_s": round(time.time() - t2, 1)}]


def main():
    which = sys.argv[1:] or ["1", "2", "3", "5"]
    info = {"gpu": torch.cuda.get_device_name(0), "lib": sc.build_info()}
    try:
        info["host_mem_gb"] = round(os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") / 1e9, 1)
    except Exception:
        pass
    print(json.dumps({"info": info}), flush=True)
    for c in which:
        fn = {"1": cfg1, "2": cfg2, "3": cfg3, "4": cfg4, "5": cfg5}[c]
        for line in fn():
            print(json.dumps(line), flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
