"""bench.py's N=1 arm: one stream resident in HBM, K timed seqcdc_chunk calls."""
from __future__ import annotations

import os
import time

import numpy as np
import torch

from .common import METRIC, ClockSampler, Workload, cpu_desc, peaks, src_hash, step_stats, traffic


class Stream:
    """A workload's stream on the device plus the call's buffers."""

    def __init__(self, w: Workload, dev):
        import synth
        import paper_2505_21194_b200 as sc
        self.w, self.dev = w, dev
        self.p = sc.SeqParams.table1(w.avg_kib, w.mode)
        if w.kind == "versions":                 # config 4: the versioned stream is built as a piece table
            self.data, _ = synth.versions_device(w.seed, 4 << 30, device=dev)
            assert self.data.numel() == w.n, (self.data.numel(), w.n)
        else:
            self.data = torch.empty(w.n, dtype=torch.uint8, device=dev)
            synth.fill_device(w.kind, w.seed, 0, self.data)
        self.cuts = torch.empty(max(sc.max_cuts(w.n, self.p), 1), dtype=torch.int64, device=dev)
        self.ncuts = torch.zeros(1, dtype=torch.int64, device=dev)
        self.ws = torch.empty(sc.workspace_size(w.n, 1, self.p), dtype=torch.uint8, device=dev)
        self.stream = torch.cuda.current_stream(dev)
        torch.cuda.synchronize()

    def step(self):
        import paper_2505_21194_b200 as sc
        sc.chunk_into(self.data, self.p, self.cuts, self.ncuts, workspace=self.ws, stream=self.stream)

    def timed(self, steps: int, warmup: int, clocks: int | None = None):
        """W untimed steps, then exactly K steps between two synchronisations,
        a CUDA-event pair around each step (on the launching stream).  Also
        returns the library's kernel launches inside the region."""
        import paper_2505_21194_b200 as sc
        for _ in range(warmup):
            self.step()
        torch.cuda.synchronize()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
        clk = ClockSampler(clocks) if clocks is not None else None
        if clk:
            clk.__enter__()
        torch.cuda.synchronize()
        l0 = sc.launch_count()
        evs[0].record(self.stream)
        for i in range(steps):
            self.step()
            evs[i + 1].record(self.stream)
        torch.cuda.synchronize()
        self.launches = sc.launch_count() - l0
        if clk:
            clk.__exit__()
        per = [evs[i].elapsed_time(evs[i + 1]) for i in range(steps)]
        return evs[0].elapsed_time(evs[-1]) / steps, per, (clk.summary() if clk else None)

    def kernel_profile(self, steps: int):
        """A second region of K steps with the library's per-phase CUDA events
        (recorded on the launching stream; they also switch off the programmatic
        launch overlap of the post kernel, so this region is slightly slower)."""
        import paper_2505_21194_b200 as sc
        sc.profile_enable(True)
        for _ in range(steps):
            self.step()
        torch.cuda.synchronize()
        prof, ncalls = sc.profile_collect()
        sc.profile_enable(False)
        return {k: v / max(ncalls, 1) for k, v in prof.items()}

    def host_cuts(self) -> np.ndarray:
        k = int(self.ncuts.item())
        return self.cuts[:k].cpu().numpy().astype(np.uint64)

    def free(self):
        del self.data, self.cuts, self.ws
        torch.cuda.empty_cache()


def _pinned_copy(t: torch.Tensor) -> torch.Tensor:
    h = torch.empty(t.numel(), dtype=torch.uint8, pin_memory=True)
    piece = 1 << 30
    for a in range(0, t.numel(), piece):
        h[a:a + piece].copy_(t[a:a + piece], non_blocking=True)
    torch.cuda.synchronize()
    return h


def e2e(st: Stream, host_in: torch.Tensor, steps: int):
    """The same metric through the public API with HOST buffers: each step copies
    the stream from pinned host memory to the device, chunks it, and reads the
    cut count and the cut list back (copies inside the timed region)."""
    host_cuts = torch.empty(st.cuts.numel(), dtype=torch.int64, pin_memory=True)
    host_n = torch.empty(1, dtype=torch.int64, pin_memory=True)
    d2h = 0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        st.data.copy_(host_in, non_blocking=True)
        st.step()
        host_n.copy_(st.ncuts, non_blocking=True)
        torch.cuda.synchronize()              # the count sizes the cut read-back
        k = int(host_n.item())
        host_cuts[:k].copy_(st.cuts[:k], non_blocking=True)
        torch.cuda.synchronize()
        d2h = 8 + 8 * k
    dt = (time.perf_counter() - t0) / steps
    return {"value": round(st.w.n / dt / 1e9, 3), "unit": "GB/s", "h2d_bytes_per_step": st.w.n,
            "d2h_bytes_per_step": d2h, "steps": steps,
            "how": "pinned host -> device copy of the stream, seqcdc_chunk, device -> host count + cut list, "
                   "per step (wall clock around synchronised steps)"}


def extra_line(w: Workload, dev, steps: int, warmup: int, walker: str | None = None) -> dict:
    """A secondary workload (not the headline): K timed calls + whole-list parity
    (`walker` forces SEQCDC_WALKER for this line)."""
    from . import verify
    import paper_2505_21194_b200 as sc
    old = os.environ.get("SEQCDC_WALKER")
    if walker:
        os.environ["SEQCDC_WALKER"] = walker
    try:
        return _extra_line(w, dev, steps, warmup) | {"walker": walker or "auto", "lib": sc.build_info()}
    finally:
        if walker:
            if old is None:
                os.environ.pop("SEQCDC_WALKER", None)
            else:
                os.environ["SEQCDC_WALKER"] = old


def _extra_line(w: Workload, dev, steps: int, warmup: int) -> dict:
    from . import verify
    st = Stream(w, dev)
    ms, per, _ = st.timed(steps, warmup)
    got = st.host_cuts()
    host = _pinned_copy(st.data).numpy()
    chk = verify.check_windows(lambda a, b: host[a:b], w.n, verify.oracle_params(w), got)
    st.free()
    gbs = w.n / ms / 1e6
    peak, _ = peaks()
    return {"workload": w.text, "stream_bytes": w.n, "value": round(gbs, 1), "unit": "GB/s",
            "ms_per_step": round(ms, 4), "step_stats": step_stats(per), "frac_of_measured_copy_peak": round(gbs / peak, 4),
            "bit_exact": chk["bit_exact"], "ncuts": int(got.size),
            "touched_fraction": chk.get("touched_fraction")}


def run(args, w: Workload) -> int:
    import paper_2505_21194_b200 as sc
    from . import verify
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    st = Stream(w, dev)
    ms, per, clocks = st.timed(args.steps, args.warmup, clocks=0)
    value = w.n / (ms / 1e3) / 1e9
    phases = st.kernel_profile(args.steps)
    lib_tag = sc.build_info()
    launches = st.launches
    if args.profile_only:
        print({"value": value, "ms": ms, "phases": phases, "lib": lib_tag}, flush=True)
        return 0
    got = st.host_cuts()
    host_t = _pinned_copy(st.data)
    ee = e2e(st, host_t, max(2, min(args.steps, 3)))
    host = host_t.numpy()
    get = lambda a, b: host[a:b]       # noqa: E731
    p_or = verify.oracle_params(w)
    chk = verify.check_windows(get, w.n, p_or, got)
    cpu1 = verify.time_oracle_single(get, w.n, p_or, got, budget_s=args.cpu_budget)
    del host_t, host
    st.free()

    peak, peak_src = peaks()
    walk_ms = phases["walk"]
    alg = chk.get("touched_bytes", {}).get("32B_units")
    achieved = alg / (walk_ms / 1e3) / 1e9 if alg else None
    kernel = "k_lwalk" if "last call: lane walker" in lib_tag else "k_walk"
    tr, tr_src = traffic(kernel, w.key)
    roof = {"bound": "hbm", "achieved": round(achieved, 1) if achieved else None, "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4) if achieved else None, "traffic": tr,
            "kernel": kernel, "kernel_ms": round(walk_ms, 4), "algorithmic_bytes": alg,
            "algorithmic_def": "32-B sectors (stream-aligned) holding a byte of a pair the method compares, counted "
                               "by the instrumented oracle over the whole stream (SURVEY.md 8(d)); the sub-minimum "
                               "and skipped regions are never read by the method (P:179, P:189)",
            "input_rate": {"GBps": round(w.n / walk_ms / 1e6, 1), "frac": round(w.n / walk_ms / 1e6 / peak, 4),
                           "def": f"stream bytes / {kernel} time (dense-equivalent rate)"},
            "dram_rate": ({"GBps": round(tr / walk_ms / 1e6, 1), "frac": round(tr / walk_ms / 1e6 / peak, 4),
                           "source": tr_src} if tr else None),
            "touched_fraction": chk.get("touched_fraction"),
            "peak_source": peak_src, "share_of_step": round(walk_ms / phases["call"], 3),
            "kernel_timing": f"CUDA events around {kernel} on the launching stream (library profile hooks), "
                             "second region of K steps"}
    extras = {}
    if not args.no_extras:
        from .common import CFG2, RAMP4G
        for ew in (CFG2, RAMP4G):
            extras[ew.key] = extra_line(ew, dev, max(5, min(args.steps, 20)), args.warmup)
        if kernel == "k_lwalk":          # the same stream on the dense warp walker, for comparison
            extras[w.key + "_warp_walker"] = extra_line(w, dev, max(5, min(args.steps, 10)), args.warmup, "warp")
    ok = chk["bit_exact"] and all(e["bit_exact"] for e in extras.values())
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic", "config": w.config(),
        "parallelism": "single GPU, segment-speculative chains, one stream",
        "step_stats": step_stats(per),
        "roofline": roof,
        "phases_ms": {k: round(v, 4) for k, v in phases.items()},
        "parity": {"vs_oracle": "whole cut list: independent oracle windows started at the GPU's own cuts "
                                "(benchlib/verify.py), all host cores", "bit_exact": chk["bit_exact"],
                   "ncuts": int(got.size), "first_mismatch": chk.get("first_mismatch"),
                   "oracle_threads": chk.get("threads"), "oracle_s": chk.get("oracle_s"),
                   "oracle_all_cores_GBps": round(w.n / chk["oracle_s"] / 1e9, 3) if chk.get("oracle_s") else None},
        "cpu_baseline": {"value": cpu1["GBps"], "unit": "GB/s", "cores": 1, "kind": "oracle",
                         "sample": f"first {cpu1['bytes']} bytes of the stream in 1 GiB pieces starting at true cuts "
                                   f"({cpu1['bytes_processed']} bytes processed incl. piece overlaps, "
                                   f"{cpu1['seconds']} s, plain single-threaded C loop)",
                         "cpu": cpu_desc(), "host_cores": os.cpu_count()},
        "e2e": ee,
        "clocks": clocks,
        "gpu_launches": launches,
        "gpu_launches_per_step": round(launches / args.steps, 2),
        "lib": lib_tag,
        "src_hash": src_hash(),
        "also": extras,
    }
    print(json_dumps(line), flush=True)
    return 0 if ok else 3


def json_dumps(x):
    import json
    return json.dumps(x)
