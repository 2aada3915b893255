"""bench.py's N>1 arm: strong scaling of ONE stream (config 5, 64 GiB) over
N ranks, one per GPU (torchrun).  Rank r holds the contiguous range
[r n/N, (r+1) n/N) plus a right halo, generated locally by the block-addressable
generator (no data-path collective); the seam protocol of
paper_2505_21194_b200/dist.py stitches the ranges (fused peer-memory exchange,
else two small all_gathers).  Timed: K steps between barrier + synchronise,
max over ranks.  Parity: every rank's list gathered to rank 0 and the
concatenation checked against the oracle over the whole stream, plus each
rank's first_index and the total."""
from __future__ import annotations

import json
import os
import time

import numpy as np
import torch
import torch.distributed as dist

from .common import METRIC, ClockSampler, Workload, cpu_desc, peaks, step_stats


def run(args, w: Workload) -> int:
    import synth
    import paper_2505_21194_b200 as sc
    from paper_2505_21194_b200.dist import CudaRangeBackend, Shard, chunk_sharded

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    # SEQCDC_DIST_BACKEND=gloo: host-side exchange, ranks may share a GPU (testing the
    # N>1 path on a one-GPU box; no kernel of one rank waits on another's)
    backend = os.environ.get("SEQCDC_DIST_BACKEND", "nccl")
    dev = torch.device("cuda", local % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group(backend)
    try:
        n = w.n
        p = sc.SeqParams.table1(w.avg_kib, w.mode)
        lo, hi = rank * n // world, (rank + 1) * n // world
        end = n if rank == world - 1 else min(n, hi + (CudaRangeBackend.TAIL + 1) * p.max_size)
        buf = torch.empty(end - lo, dtype=torch.uint8, device=dev)
        synth.fill_device(w.kind, w.seed, lo, buf)
        shard = Shard(buf, hi - lo, lo, n)
        be = CudaRangeBackend(p, device=dev)
        exchange = os.environ.get("SEQCDC_EXCHANGE", "p2p")
        if exchange == "p2p" and not be.enable_p2p():
            exchange = f"collective (p2p unavailable: {be.p2p_error})"
        stream = torch.cuda.current_stream(dev)
        torch.cuda.synchronize()
        for _ in range(args.warmup):
            res = chunk_sharded(shard, be)
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
        with ClockSampler(local) as clk:
            dist.barrier()
            torch.cuda.synchronize()
            l0 = sc.launch_count()
            evs[0].record(stream)
            for i in range(args.steps):
                res = chunk_sharded(shard, be)
                evs[i + 1].record(stream)
            torch.cuda.synchronize()
            nl = sc.launch_count() - l0
            dist.barrier()
        per_local = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]
        t = torch.tensor([evs[0].elapsed_time(evs[-1]) / args.steps] + per_local, dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0].item())
        tl = torch.tensor([nl], dtype=torch.int64, device=dev)
        dist.all_reduce(tl)                    # launches summed over ranks
        per = t[1:].tolist()                  # per step: max over ranks
        value = n / (ms / 1e3) / 1e9
        path = be.last_path

        # end to end: each rank's pinned host shard -> device, sharded chunking, cuts -> host
        host_in = torch.empty(buf.numel(), dtype=torch.uint8, pin_memory=True)
        host_in.copy_(buf)                    # device -> pinned host directly (no pageable copy of the shard)
        torch.cuda.synchronize()
        host_cuts = torch.empty(be.out_cuts.numel(), dtype=torch.int64, pin_memory=True)
        e2e_steps = max(2, min(args.steps, 3))
        d2h = 0
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            buf.copy_(host_in, non_blocking=True)
            r2 = chunk_sharded(shard, be)
            host_cuts[: r2.count].copy_(r2.cuts[: r2.count], non_blocking=True)
            torch.cuda.synchronize()
            d2h = 8 * r2.count
        te = torch.tensor([(time.perf_counter() - t0) / e2e_steps], dtype=torch.float64, device=dev)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_value = n / float(te.item()) / 1e9
        del host_in

        # parity: gather every rank's list, check the concatenation on rank 0
        mine = res.cuts[: res.count].cpu().numpy().astype(np.uint64)
        meta = [res.first_index, res.count, res.total]
        lists = [None] * world if rank == 0 else None
        metas = [None] * world if rank == 0 else None
        dist.gather_object(mine, lists, dst=0)
        dist.gather_object(meta, metas, dst=0)
        be.close()
        if rank != 0:
            dist.barrier()
            return 0
        from . import verify
        allc = np.concatenate(lists) if lists else np.zeros(0, np.uint64)
        idx_ok = all(metas[r][0] == sum(m[1] for m in metas[:r]) for r in range(world)) and \
            all(m[2] == allc.size for m in metas)

        def get(a, b):
            return synth.fill_host(w.kind, w.seed, a, b - a)
        chk = verify.check_windows(get, n, verify.oracle_params(w), allc)
        dist.barrier()
        peak, peak_src = peaks()
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic", "config": w.config(),
            "parallelism": f"{world} ranks x contiguous {n // world}-byte ranges of one stream, seam exchange: "
                           f"{exchange}, last step's path: {path}",
            "step_stats": step_stats(per),
            "per_gpu_input_GBps": round(value / world, 1),
            "parity": {"vs_oracle": "concatenated rank lists vs the oracle over the whole stream (bytes regenerated "
                                    "on the host), plus every rank's first_index and the total",
                       "bit_exact": bool(chk["bit_exact"] and idx_ok), "lists_equal": chk["bit_exact"],
                       "first_index_and_total_ok": idx_ok, "ncuts": int(allc.size),
                       "first_mismatch": chk.get("first_mismatch"), "oracle_threads": chk.get("threads"),
                       "oracle_s": chk.get("oracle_s")},
            "roofline": {"bound": "hbm", "peak": peak, "peak_source": peak_src, "unit": "GB/s",
                         "algorithmic_bytes": chk.get("touched_bytes", {}).get("32B_units"),
                         "achieved_per_gpu": (round(chk["touched_bytes"]["32B_units"] / world / ms / 1e6, 1)
                                              if chk.get("touched_bytes") else None),
                         "note": "per-GPU algorithmic bytes / step time (whole step, incl. the seam exchange)"},
            "e2e": {"value": round(e2e_value, 3), "unit": "GB/s", "h2d_bytes_per_step": n,
                    "d2h_bytes_per_step": d2h * world,
                    "how": "every rank: pinned host range -> device, sharded chunking, its cuts -> host; max over ranks"},
            "clocks": clk.summary(),
            "gpu_launches": int(tl.item()),
            "cpu": cpu_desc(),
        }
        print(json.dumps(line), flush=True)
        return 0 if line["parity"]["bit_exact"] else 3
    finally:
        dist.destroy_process_group()
