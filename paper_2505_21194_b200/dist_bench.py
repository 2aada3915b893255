"""bench.py's N>1 arm: one stream of N x bytes_per_gpu bytes sharded into
contiguous ranges, one rank per GPU (torchrun), NCCL for the two small
exchanges of the sharded protocol (dist.py).  Weak scaling: every rank holds
bytes_per_gpu bytes of the stream plus a max_size halo, generated locally by
the block-addressable generators (no data-path collective)."""
from __future__ import annotations

import json
import os
import time

import numpy as np
import torch
import torch.distributed as dist


def run(args, metric, workload, cfg):
    import synth
    import paper_2505_21194_b200 as sc
    from .dist import CudaRangeBackend, Shard, chunk_sharded

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    # SEQCDC_DIST_BACKEND=gloo: host-side exchange, ranks may share a GPU (testing the
    # N>1 path on a single-GPU box; kernels of different ranks never wait on each other)
    backend = os.environ.get("SEQCDC_DIST_BACKEND", "nccl")
    dev = torch.device("cuda", local % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=dev)
        cdev = dev
    else:
        dist.init_process_group(backend)
        cdev = dev                      # gloo handles CUDA tensors too: same device protocol as NCCL
    try:
        n_per = args.bytes_per_gpu
        n = n_per * world
        p = sc.SeqParams.table1(cfg["avg_kib"], cfg["mode"])
        lo, hi = rank * n_per, (rank + 1) * n_per
        # halo: room for the range's tail continuation (device protocol, dist.py)
        end = n if rank == world - 1 else min(n, hi + (CudaRangeBackend.TAIL + 1) * p.max_size)
        buf = torch.empty(end - lo, dtype=torch.uint8, device=dev)
        synth.fill_device(cfg["kind"], cfg["seed"], lo, buf)
        shard = Shard(buf, hi - lo, lo)
        be = CudaRangeBackend(p, device=dev)
        be.comm_device = cdev
        # SEQCDC_EXCHANGE=p2p (default): fused exchange over peer memory (the range's
        # last kernel stores its block into the next rank's mailbox); "collective":
        # NCCL/gloo all_gather of the blocks
        exchange = os.environ.get("SEQCDC_EXCHANGE", "p2p")
        if exchange == "p2p" and world > 1 and not be.enable_p2p():
            exchange = f"collective (p2p unavailable: {be.p2p_error})"
        exchange = exchange if world > 1 else "none"
        stream = torch.cuda.current_stream(dev)
        torch.cuda.synchronize()
        for _ in range(args.warmup):
            res = chunk_sharded(shard, be)
        from bench import ClockSampler, _peaks, _cpu_desc, time_oracle
        sc.profile_enable(True)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as clk:
            dist.barrier()
            torch.cuda.synchronize()
            ev0.record(stream)
            for _ in range(args.steps):
                res = chunk_sharded(shard, be)
            ev1.record(stream)
            torch.cuda.synchronize()
            dist.barrier()
        prof, ncalls = sc.profile_collect()
        sc.profile_enable(False)
        ms_local = ev0.elapsed_time(ev1) / args.steps
        t = torch.tensor([ms_local], dtype=torch.float64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        value = n / (ms / 1e3) / 1e9
        walk_ms = prof["walk"] / max(ncalls, 1)

        # end to end: pinned host shard -> device, sharded chunking, cuts -> host
        host_in = torch.empty(buf.numel(), dtype=torch.uint8, pin_memory=True)
        host_in.copy_(buf.cpu())
        host_cuts = torch.empty(be.out_cuts.numel(), dtype=torch.int64, pin_memory=True)
        e2e_steps = max(2, min(args.steps, 5))
        d2h = 0
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            buf.copy_(host_in, non_blocking=True)
            r2 = chunk_sharded(shard, be)
            host_cuts[: r2.count].copy_(r2.cuts[: r2.count], non_blocking=True)
            torch.cuda.synchronize()
            d2h = 8 * r2.count
        e2e_local = (time.perf_counter() - t0) / e2e_steps
        t = torch.tensor([e2e_local], dtype=torch.float64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_value = n / float(t.item()) / 1e9

        # parity: each rank's chain re-derived by the oracle from its true entry
        import oracle
        op = oracle.table1(cfg["avg_kib"], cfg["mode"])
        hb = host_in.numpy()
        sub = oracle.chunk(hb[res.entry - lo:], op)
        sub = sub + np.uint64(res.entry)
        k_end = int(np.searchsorted(sub, np.uint64(hi), side="left"))
        want = sub[: k_end + 1] if rank < world - 1 else sub
        got = res.cuts[: res.count].cpu().numpy().astype(np.uint64)
        ok = torch.tensor([1 if (got.size == want.size and np.array_equal(got, want)) else 0], device=cdev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        exact = bool(ok.item())

        if rank == 0:
            cpu_value, passes, cpu_t, _ = time_oracle(hb[:n_per], budget_s=8.0, max_passes=2)
            peak, peak_src = _peaks()
            line = {
                "metric": metric, "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "u8", "data": "synthetic",
                "config": {"workload": workload + f"; one stream of {world} x {n_per} bytes, contiguous ranges",
                           "stream_bytes": n, "bytes_per_gpu": n_per,
                           "parallelism": f"{world} contiguous ranges + seam exchange (dist.py)",
                           "exchange": exchange, "last_round": getattr(be, "last_path", None),
                           "l2": "input per GPU > 126 MB L2: no flush needed", "ncuts": res.total,
                           "resync_rounds": res.rounds, "dist_backend": backend},
                "roofline": {"bound": "hbm", "achieved": round(n_per / (walk_ms / 1e3) / 1e9, 1), "peak": peak,
                             "unit": "GB/s", "frac": round(n_per / (walk_ms / 1e3) / 1e9 / peak, 4), "traffic": None,
                             "kernel": "k_walk", "kernel_ms": round(walk_ms, 4), "peak_source": peak_src},
                "cpu_baseline": {"value": round(cpu_value, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
                                 "sample": f"rank 0's {n_per}-byte range x{passes} passes ({cpu_t:.1f} s)",
                                 "cpu": _cpu_desc(), "host_cores": os.cpu_count()},
                "e2e": {"value": round(e2e_value, 3), "unit": "GB/s", "h2d_bytes_per_step": int(buf.numel()) * world,
                        "d2h_bytes_per_step": d2h * world},
                "clocks": clk.summary(),
                "gpu_launches": (7 + 2) * args.steps,
                "parity": {"vs_oracle": "every rank's whole cut list (oracle from its true entry)", "bit_exact": exact},
            }
            print(json.dumps(line), flush=True)
        dist.barrier()                     # no rank still uses a peer mailbox
        be.close()
        return 0 if exact else 3
    finally:
        dist.destroy_process_group()
