"""Workload definitions, peaks, clock sampling and host facts for bench.py."""
from __future__ import annotations

import json
import os
import platform
import threading
import time
from dataclasses import dataclass

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRIC = "SeqCDC chunking GB/s at 1/2/4/8 B200; % of HBM-read roofline; cuts bit-exact"
GiB, MiB = 1 << 30, 1 << 20


@dataclass(frozen=True)
class Workload:
    """One BASELINE.json config as a synthetic stream (synth/) + SeqCDC parameters
    (Table I row, min = avg/2, max = 2 avg; readings c11/c12)."""

    key: str
    text: str
    kind: str
    seed: int
    n: int
    avg_kib: int
    mode: int

    def config(self) -> dict:
        """The `config` object of the bench line (identical in both arms)."""
        L, T, S = {4: (5, 55, 256), 8: (5, 50, 256), 16: (5, 50, 512)}[self.avg_kib]
        return {"workload": self.text, "stream_bytes": self.n, "generator": f"{self.kind} seed {self.seed}",
                "params": {"mode": "Decreasing" if self.mode else "Increasing", "seq_length": L,
                           "skip_trigger": T, "skip_size": S, "min_size": self.avg_kib * 512,
                           "max_size": self.avg_kib * 2048},
                "l2": f"input {self.n / GiB:.3g} GiB > 126 MB L2: no flush needed between steps"}

    def resized(self, n: int) -> "Workload":
        return Workload(self.key, self.text + f" [resized to {n} bytes]", self.kind, self.seed, n, self.avg_kib,
                        self.mode)


CFG5 = Workload("cfg5", "config 5: one 64 GiB stream, 50/50 uniform random bytes and +-1 byte ramps of random length "
                "2-600 (rampmix seed 5); Increasing, SeqLength 5, SkipTrigger 50, SkipSize 256, min 4 KiB, max 16 KiB; "
                "sharded over N GPUs (strong scaling)", "rampmix", 5, 64 * GiB, 8, 0)
CFG2 = Workload("cfg2", "config 2: 1 GiB order-1 Markov text (seed 2); Decreasing, SeqLength 5, SkipTrigger 55, "
                "SkipSize 256, min 2 KiB, max 8 KiB", "markov", 2, GiB, 4, 1)
RAMP4G = Workload("rampmix4g", "north-star line: 4 GiB + 12345 B of the config-5 generator; Increasing, L5 T50 S256, "
                  "min 4 KiB, max 16 KiB", "rampmix", 5, 4 * GiB + 12345, 8, 0)
CFG4 = Workload("cfg4", "config 4: versioned backup stream, 4 GiB uniform base + 10 versions with seeded 1% edits "
                "(inserts/deletes/overwrites of 1 B-4 KiB), ~44 GiB, one stream; Increasing, SeqLength 5, SkipTrigger 50, "
                "SkipSize 512, min 8 KiB, max 32 KiB", "versions", 4, 47240893232, 16, 0)
WORKLOADS = {w.key: w for w in (CFG5, CFG2, RAMP4G, CFG4)}


def peaks():
    """(HBM GB/s, source): MEASURED_PEAKS.json's copy figure, else the profiling
    guide's fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def src_hash() -> str:
    """Hash of the library's sources (csrc/ + include/): identifies the build an
    ncu capture was taken with."""
    import hashlib
    h = hashlib.sha256()
    for d in (os.path.join(ROOT, "paper_2505_21194_b200", "csrc"), os.path.join(ROOT, "include")):
        for f in sorted(os.listdir(d)):
            if f.endswith((".cu", ".cuh", ".h")):
                with open(os.path.join(d, f), "rb") as fh:
                    h.update(f.encode() + fh.read())
    return h.hexdigest()[:16]


def traffic(kernel: str, workload_key: str):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full capture
    (profiles/traffic.json), if it was taken on this workload with these sources."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            d = json.load(f)[f"{kernel}:{workload_key}"]
        if d.get("src_hash") != src_hash():
            return None, None
        return int(d["dram_read_bytes"]) + int(d["dram_write_bytes"]), d.get("source")
    except Exception:
        return None, None


def cpu_desc():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor()


class ClockSampler:
    """nvidia-smi-equivalent (NVML) SM clock and throttle-reason samples taken
    DURING the timed region."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks",
               0x1: "gpu_idle", 0x10: "sync_boost"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self._nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._nv:
            self._t.join()

    def summary(self):
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2] if s else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(s)}


def step_stats(ms_list):
    s = sorted(ms_list)
    return {"median_ms": round(s[len(s) // 2], 4), "best_ms": round(s[0], 4),
            "mean_ms": round(sum(s) / len(s), 4), "worst_ms": round(s[-1], 4), "regions": len(s),
            "how": "one CUDA-event pair around each timed step (each step one region)"}
