#!/usr/bin/env python
"""Summarise an ncu report / launch list for profiles/ (run here, no GPU needed).

  python tools/ncu_summary.py report.ncu-rep [--sass N]   -> key metrics, stall mix, hot SASS
  python tools/ncu_summary.py launches.csv                -> per-kernel mean durations and shares
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum.per_second",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size",
        "launch__occupancy_limit_shared_mem", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__inst_executed_pipe_alu.sum", "smsp__inst_executed_pipe_fma.sum",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_uniform.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "lts__t_requests_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
        "lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum", "lts__t_sectors.sum"]


def report(path, nsass=0):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print(f"## kernel: {name}")
        for i, k in enumerate(h):
            if k in KEYS:
                print(f"  {k:70s} {r[i]:>18s} {u[i]}")
        st = []
        for i, k in enumerate(h):
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    st.append((float(r[i].replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(x for x, _ in st) or 1
        print("  stall samples (share):", ", ".join(f"{n} {x / tot:.1%}" for x, n in sorted(st, reverse=True)[:9]))

        def g(k):
            try:
                return float(r[h.index(k)].replace(",", ""))
            except (ValueError, IndexError):
                return None
        req, sec = g("lts__t_requests_srcunit_tex_op_read.sum"), g("lts__t_sectors_srcunit_tex_op_read.sum")
        hit = g("lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum")
        if req and sec:
            print(f"  L2 read sectors per request (from L1/TEX): {sec / req:.2f} (4.00 = full 128-B lines); "
                  f"L2 read hit rate {hit / sec:.1%}" if hit is not None else "")
    if nsass:
        src = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                             capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(src)))
        h = rows[1]
        ia, isrc, iss, iex = (h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"),
                              h.index("Instructions Executed"))
        data = []
        for r in rows[2:]:
            try:
                data.append((r[ia], r[isrc], float(r[iss] or 0), float(r[iex] or 0)))
            except (ValueError, IndexError):
                pass
        print(f"  top {nsass} SASS by stall samples:")
        for a, s, ss, ex in sorted(data, key=lambda d: -d[2])[:nsass]:
            print(f"    {ss:7.0f} {ex:12.0f}  {s[:90]}")


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ik, iv = h.index("Kernel Name"), h.index("Metric Value")
    d = defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > iv:
            d[r[ik].split("(")[0][:60]].append(float(r[iv].replace(",", "")) / 1e3)
    print(f"{'kernel':62s} {'n':>4s} {'mean us':>10s} {'min us':>10s}")
    for k, v in d.items():
        print(f"{k:62s} {len(v):4d} {sum(v) / len(v):10.1f} {min(v):10.1f}")


if __name__ == "__main__":
    p = sys.argv[1]
    if p.endswith(".csv"):
        launches(p)
    else:
        report(p, int(sys.argv[sys.argv.index("--sass") + 1]) if "--sass" in sys.argv else 0)
