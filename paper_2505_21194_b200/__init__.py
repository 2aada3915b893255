"""B200-native SeqCDC boundary detection (arXiv 2505.21194) -- Python binding.

Thin ctypes binding over the C ABI in ``include/seqcdc.h`` (libseqcdc.so,
built in-tree from ``csrc/``).  Argument marshalling only: every step of the
chunking path runs in the library's CUDA kernels.  PyTorch supplies device
memory and streams.  There is no CPU fallback: if the extension is missing or
no CUDA device is present, calls raise.

Names follow the paper: ``mode`` (Increasing/Decreasing),
``seq_length`` (SeqLength), ``skip_trigger`` (SkipTrigger), ``skip_size``
(SkipSize), ``min_size``/``max_size``.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

from . import _build

INCREASING = 0
DECREASING = 1
FLAG_SIGNED = 1
FLAG_PAIRS = 2      # SeqLength counts favourable comparisons (reading c1's alternative)

SEQCDC_OK, SEQCDC_EINVAL, SEQCDC_ENOMEM, SEQCDC_ECUDA = 0, 1, 2, 3
NCUTS_BAD_INPUT = (1 << 64) - 1

# Every symbol include/seqcdc.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "seqcdc_validate_params", "seqcdc_default_params", "seqcdc_max_cuts", "seqcdc_max_cuts_batch",
    "seqcdc_workspace_size", "seqcdc_chunk", "seqcdc_chunk_batch", "seqcdc_strerror",
    "seqcdc_build_info", "seqcdc_set_segment_bytes", "seqcdc_profile_enable", "seqcdc_profile_collect",
    "seqcdc_range_max_cuts", "seqcdc_range_chunk", "seqcdc_range_resync", "seqcdc_range_resync_dev",
    "seqcdc_range_chunk_tail", "seqcdc_range_merge_tail",
    "seqcdc_xchg_alloc", "seqcdc_xchg_open", "seqcdc_xchg_close", "seqcdc_xchg_free",
    "seqcdc_range_chunk_tail_push", "seqcdc_range_merge_tail_wait", "seqcdc_xchg_put_rows", "seqcdc_xchg_wait_rows",
    "seqcdc_fingerprint", "seqcdc_dedup_workspace_size", "seqcdc_dedup", "seqcdc_launch_count",
)


class _CParams(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_uint32), ("seq_length", ctypes.c_uint32),
                ("skip_trigger", ctypes.c_uint32), ("skip_size", ctypes.c_uint32),
                ("min_size", ctypes.c_uint64), ("max_size", ctypes.c_uint64),
                ("flags", ctypes.c_uint32), ("reserved", ctypes.c_uint32)]


@dataclass(frozen=True)
class SeqParams:
    """SeqCDC parameters (Table I)."""

    mode: int = INCREASING
    seq_length: int = 5
    skip_trigger: int = 50
    skip_size: int = 256
    min_size: int = 4096
    max_size: int = 16384
    flags: int = 0          # SEQCDC_FLAG_SIGNED (1): int8 byte order; SEQCDC_FLAG_PAIRS (2): L comparisons

    def c(self) -> _CParams:
        return _CParams(self.mode, self.seq_length, self.skip_trigger, self.skip_size,
                        self.min_size, self.max_size, self.flags, 0)

    @staticmethod
    def table1(avg_kib: int, mode: int = INCREASING) -> "SeqParams":
        cp = _CParams()
        _check(lib().seqcdc_default_params(avg_kib, mode, ctypes.byref(cp)), "seqcdc_default_params")
        return SeqParams(cp.mode, cp.seq_length, cp.skip_trigger, cp.skip_size, cp.min_size, cp.max_size)


class SeqCDCError(RuntimeError):
    pass


_lib = None


def lib():
    """Load libseqcdc.so (building it in-tree first if sources are newer)."""
    global _lib
    if _lib is None:
        path = os.environ.get("SEQCDC_LIB") or _build.LIB   # SEQCDC_LIB: tuning variants only
        if path == _build.LIB and _build.stale():
            path = _build.build()
        if not os.path.exists(path):
            raise SeqCDCError(f"libseqcdc.so missing at {path}; run __graft_entry__.build()")
        L = ctypes.CDLL(path)
        missing = [name for name in EXPORTS if not hasattr(L, name)]
        if missing:                      # e.g. a stale tuning build: fail now, not in a subprocess later
            raise SeqCDCError(f"{path} lacks {', '.join(missing)}: rebuild it (__graft_entry__.build() or "
                              f"tools/variants.sh)")
        u32, u64, p, sz = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_size_t
        P = ctypes.POINTER(_CParams)
        L.seqcdc_validate_params.argtypes = [P]
        L.seqcdc_validate_params.restype = ctypes.c_int
        L.seqcdc_default_params.argtypes = [u32, u32, P]
        L.seqcdc_default_params.restype = ctypes.c_int
        L.seqcdc_max_cuts.argtypes = [u64, P]
        L.seqcdc_max_cuts.restype = u64
        L.seqcdc_max_cuts_batch.argtypes = [u64, u32, P]
        L.seqcdc_max_cuts_batch.restype = u64
        L.seqcdc_workspace_size.argtypes = [u64, u32, P]
        L.seqcdc_workspace_size.restype = sz
        L.seqcdc_chunk.argtypes = [p, u64, P, p, p, p, sz, p]
        L.seqcdc_chunk.restype = ctypes.c_int
        L.seqcdc_chunk_batch.argtypes = [p, p, u32, u64, P, p, p, p, p, sz, p]
        L.seqcdc_chunk_batch.restype = ctypes.c_int
        L.seqcdc_strerror.argtypes = [ctypes.c_int]
        L.seqcdc_strerror.restype = ctypes.c_char_p
        L.seqcdc_build_info.argtypes = []
        L.seqcdc_build_info.restype = ctypes.c_char_p
        L.seqcdc_set_segment_bytes.argtypes = [u64]
        L.seqcdc_set_segment_bytes.restype = ctypes.c_int
        L.seqcdc_launch_count.argtypes = []
        L.seqcdc_launch_count.restype = u64
        L.seqcdc_profile_enable.argtypes = [ctypes.c_int]
        L.seqcdc_profile_enable.restype = ctypes.c_int
        L.seqcdc_profile_collect.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(u64)]
        L.seqcdc_profile_collect.restype = ctypes.c_int
        L.seqcdc_range_max_cuts.argtypes = [u64, u64, P]
        L.seqcdc_range_max_cuts.restype = u64
        L.seqcdc_range_chunk.argtypes = [p, u64, u64, u64, u64, P, p, p, p, sz, p]
        L.seqcdc_range_chunk.restype = ctypes.c_int
        L.seqcdc_range_resync.argtypes = [p, u64, u64, u64, u64, P, p, p, p, p, p, p]
        L.seqcdc_range_resync.restype = ctypes.c_int
        L.seqcdc_range_resync_dev.argtypes = [p, u64, u64, p, u64, P, p, p, p, p, p, p]
        L.seqcdc_range_resync_dev.restype = ctypes.c_int
        L.seqcdc_range_chunk_tail.argtypes = [p, u64, u64, u64, u64, P, p, p, u32, p, p, p, p, sz, p]
        L.seqcdc_range_chunk_tail.restype = ctypes.c_int
        L.seqcdc_range_merge_tail.argtypes = [p, u64, u64, u64, P, p, u32, p, p, p, p, p, p, p, p]
        L.seqcdc_range_merge_tail.restype = ctypes.c_int
        L.seqcdc_xchg_alloc.argtypes = [sz, ctypes.POINTER(p), p]
        L.seqcdc_xchg_alloc.restype = ctypes.c_int
        L.seqcdc_xchg_open.argtypes = [p, ctypes.POINTER(p)]
        L.seqcdc_xchg_open.restype = ctypes.c_int
        L.seqcdc_xchg_close.argtypes = [p]
        L.seqcdc_xchg_close.restype = ctypes.c_int
        L.seqcdc_xchg_free.argtypes = [p]
        L.seqcdc_xchg_free.restype = ctypes.c_int
        L.seqcdc_range_chunk_tail_push.argtypes = [p, u64, u64, u64, u64, P, p, p, u32, p, p, p, p, sz, p, p, u64, p]
        L.seqcdc_range_chunk_tail_push.restype = ctypes.c_int
        L.seqcdc_range_merge_tail_wait.argtypes = [p, u64, u64, u64, P, p, u32, p, p, p, p, p, p, p, p, u64, u64, p]
        L.seqcdc_range_merge_tail_wait.restype = ctypes.c_int
        L.seqcdc_xchg_put_rows.argtypes = [p, u32, p, u32, u32, u64, p]
        L.seqcdc_xchg_put_rows.restype = ctypes.c_int
        L.seqcdc_xchg_wait_rows.argtypes = [p, u32, u32, u64, u64, p, p, p]
        L.seqcdc_xchg_wait_rows.restype = ctypes.c_int
        L.seqcdc_fingerprint.argtypes = [p, p, p, u64, p, p]
        L.seqcdc_fingerprint.restype = ctypes.c_int
        L.seqcdc_dedup_workspace_size.argtypes = [u64]
        L.seqcdc_dedup_workspace_size.restype = sz
        L.seqcdc_dedup.argtypes = [p, p, p, u64, p, p, p, sz, p]
        L.seqcdc_dedup.restype = ctypes.c_int
        _lib = L
    return _lib


def _check(rc: int, what: str) -> None:
    if rc != SEQCDC_OK:
        raise SeqCDCError(f"{what}: {lib().seqcdc_strerror(rc).decode()} ({rc})")


def validate(p: SeqParams) -> bool:
    cp = p.c()
    return lib().seqcdc_validate_params(ctypes.byref(cp)) == SEQCDC_OK


def max_cuts(n: int, p: SeqParams) -> int:
    cp = p.c()
    return int(lib().seqcdc_max_cuts(n, ctypes.byref(cp)))


def max_cuts_batch(total: int, nstreams: int, p: SeqParams) -> int:
    cp = p.c()
    return int(lib().seqcdc_max_cuts_batch(total, nstreams, ctypes.byref(cp)))


def workspace_size(total: int, nstreams: int, p: SeqParams) -> int:
    cp = p.c()
    return int(lib().seqcdc_workspace_size(total, nstreams, ctypes.byref(cp)))


def set_segment_bytes(g: int) -> None:
    """Force the speculative segment length (testing/tuning); 0 = automatic."""
    _check(lib().seqcdc_set_segment_bytes(int(g)), "seqcdc_set_segment_bytes")


def profile_enable(on: bool = True) -> None:
    _check(lib().seqcdc_profile_enable(1 if on else 0), "seqcdc_profile_enable")


def profile_collect():
    """-> (dict of summed ms per phase, number of calls) since profile_enable()."""
    ms = (ctypes.c_double * 4)()
    n = ctypes.c_uint64(0)
    _check(lib().seqcdc_profile_collect(ms, ctypes.byref(n)), "seqcdc_profile_collect")
    return {"setup": ms[0], "walk": ms[1], "post": ms[2], "call": ms[3]}, int(n.value)


def launch_count() -> int:
    """Kernels the library has launched in this process so far (monotone)."""
    return int(lib().seqcdc_launch_count())


def build_info() -> str:
    return lib().seqcdc_build_info().decode()


def _stream_ptr(stream, device):
    import torch
    s = torch.cuda.current_stream(device) if stream is None else stream
    return s.cuda_stream


def _require_cuda(t, name):
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda):
        raise SeqCDCError(f"{name} must be a CUDA tensor (there is no CPU path)")
    if not t.is_contiguous():
        raise SeqCDCError(f"{name} must be contiguous")


def _require_out(t, name, min_numel: int, like, dtype=None):
    """An output/input tensor the device writes or reads by count: CUDA,
    contiguous, on `like`'s device, of `dtype` (int64 by default) and with at
    least `min_numel` elements -- the C ABI takes no capacities, so an
    undersized tensor is refused here instead of being overrun on the device."""
    import torch
    _require_cuda(t, name)
    if t.device != like.device:
        raise SeqCDCError(f"{name} is on {t.device}, the data on {like.device}")
    if t.dtype != (dtype or torch.int64):
        raise SeqCDCError(f"{name} must be {dtype or torch.int64}, got {t.dtype}")
    if t.numel() < min_numel:
        raise SeqCDCError(f"{name} holds {t.numel()} elements, needs >= {min_numel}")


def _on(t):
    """Run a library call with t's device current (kernels, pool and stream agree)."""
    import torch
    return torch.cuda.device(t.device)


def chunk_into(data, p: SeqParams, cuts, ncuts, workspace=None, stream=None) -> None:
    """Asynchronous: enqueue seqcdc_chunk on ``stream``.  ``data`` uint8 CUDA,
    ``cuts`` int64 CUDA with >= max_cuts(n) entries, ``ncuts`` int64 CUDA [1]."""
    import torch
    _require_cuda(data, "data")
    if data.dtype != torch.uint8:
        raise SeqCDCError("data must be uint8")
    n = data.numel()
    _require_out(cuts, "cuts", max_cuts(n, p), data)
    _require_out(ncuts, "ncuts", 1, data)
    if workspace is not None:
        _require_out(workspace, "workspace", 0, data, torch.uint8)
    cp = p.c()
    ws_ptr, ws_len = (workspace.data_ptr(), workspace.numel()) if workspace is not None else (None, 0)
    with _on(data):
        rc = lib().seqcdc_chunk(data.data_ptr() if n else None, n, ctypes.byref(cp),
                                cuts.data_ptr() if cuts.numel() else None, ncuts.data_ptr(), ws_ptr, ws_len,
                                _stream_ptr(stream, data.device))
    _check(rc, "seqcdc_chunk")


def chunk(data, p: SeqParams, stream=None):
    """Cut offsets (int64 CUDA tensor) of one stream.  Synchronises to size the result."""
    import torch
    _require_cuda(data, "data")
    n = data.numel()
    cuts = torch.empty(max(max_cuts(n, p), 1), dtype=torch.int64, device=data.device)
    ncuts = torch.zeros(1, dtype=torch.int64, device=data.device)
    chunk_into(data, p, cuts, ncuts, stream=stream)
    k = int(ncuts.item())
    return cuts[:k]


def chunk_batch_into(data, offsets, p: SeqParams, cuts, cut_index, ncuts, total=None, workspace=None,
                     stream=None) -> None:
    """Asynchronous batch call.  ``offsets`` int64 CUDA [ns+1]; cuts are absolute offsets into data."""
    import torch
    _require_cuda(data, "data")
    _require_cuda(offsets, "offsets")
    ns = offsets.numel() - 1
    if total is None:
        total = int(offsets[-1].item() - offsets[0].item())
    _require_out(offsets, "offsets", 1, data)
    _require_out(cuts, "cuts", max_cuts_batch(total, ns, p), data)
    _require_out(cut_index, "cut_index", ns + 1, data)
    _require_out(ncuts, "ncuts", 1, data)
    cp = p.c()
    ws_ptr, ws_len = (workspace.data_ptr(), workspace.numel()) if workspace is not None else (None, 0)
    with _on(data):
        rc = lib().seqcdc_chunk_batch(data.data_ptr() if data.numel() else None, offsets.data_ptr(), ns, total,
                                      ctypes.byref(cp), cuts.data_ptr() if cuts.numel() else None,
                                      cut_index.data_ptr(), ncuts.data_ptr(), ws_ptr, ws_len,
                                      _stream_ptr(stream, data.device))
    _check(rc, "seqcdc_chunk_batch")


def chunk_batch(data, offsets, p: SeqParams, stream=None):
    """Independent streams data[offsets[j]:offsets[j+1]] -> (cuts, cut_index), int64 CUDA tensors."""
    import torch
    ns = offsets.numel() - 1
    total = int(offsets[-1].item() - offsets[0].item())
    cuts = torch.empty(max(max_cuts_batch(total, ns, p), 1), dtype=torch.int64, device=data.device)
    cut_index = torch.empty(ns + 1, dtype=torch.int64, device=data.device)
    ncuts = torch.zeros(1, dtype=torch.int64, device=data.device)
    chunk_batch_into(data, offsets, p, cuts, cut_index, ncuts, total=total, stream=stream)
    k = int(ncuts.item())
    if k == NCUTS_BAD_INPUT - (1 << 64):
        raise SeqCDCError("inconsistent batch offsets")
    return cuts[:k], cut_index


# ------------------------------------------------------------------ range calls (multi-GPU building blocks)
def range_max_cuts(buf_len: int, range_len: int, p: SeqParams) -> int:
    cp = p.c()
    return int(lib().seqcdc_range_max_cuts(buf_len, range_len, ctypes.byref(cp)))


def range_chunk_into(buf, range_len: int, entry: int, global_offset: int, p: SeqParams, cuts, ncuts,
                     workspace=None, stream=None) -> None:
    """Asynchronous seqcdc_range_chunk: the chain from local ``entry`` up to its
    first cut >= range_len, as global offsets, into ``cuts`` / ``ncuts``."""
    import torch
    _require_cuda(buf, "buf")
    if buf.dtype != torch.uint8:
        raise SeqCDCError("buf must be uint8")
    _require_out(cuts, "cuts", range_max_cuts(buf.numel(), range_len, p), buf)
    _require_out(ncuts, "ncuts", 1, buf)
    cp = p.c()
    ws_ptr, ws_len = (workspace.data_ptr(), workspace.numel()) if workspace is not None else (None, 0)
    with _on(buf):
        rc = lib().seqcdc_range_chunk(buf.data_ptr() if buf.numel() else None, buf.numel(), range_len, entry,
                                      global_offset, ctypes.byref(cp), cuts.data_ptr() if cuts.numel() else None,
                                      ncuts.data_ptr(), ws_ptr, ws_len, _stream_ptr(stream, buf.device))
    _check(rc, "seqcdc_range_chunk")


def range_resync_into(buf, range_len: int, entry: int, global_offset: int, p: SeqParams, spec, spec_n, cuts,
                      ncuts, status, stream=None) -> None:
    """Asynchronous seqcdc_range_resync: the true chain from the true entry,
    re-using the speculative chain ``spec[:spec_n]`` after the first common cut.
    ``status`` int64 CUDA [4] = merged, re-walked cuts, merge index, overhang."""
    _require_cuda(buf, "buf")
    _require_out(cuts, "cuts", range_max_cuts(buf.numel(), range_len, p), buf)
    _require_out(status, "status", 4, buf)
    cp = p.c()
    rc = lib().seqcdc_range_resync(buf.data_ptr() if buf.numel() else None, buf.numel(), range_len, entry,
                                   global_offset, ctypes.byref(cp), spec.data_ptr() if spec.numel() else None,
                                   spec_n.data_ptr(), cuts.data_ptr() if cuts.numel() else None, ncuts.data_ptr(),
                                   status.data_ptr(), _stream_ptr(stream, buf.device))
    _check(rc, "seqcdc_range_resync")


# ------------------------------------------------------------------ after chunking: fingerprints + dedup (NEXT-1)
def fingerprint_into(data, cuts, ncuts, digests, max_cuts=None, stream=None) -> None:
    """Asynchronous seqcdc_fingerprint: SHA-256 of every chunk into ``digests``
    (uint8 CUDA [>= 32*max_cuts], 16-byte aligned); the count is read from ``ncuts``."""
    _require_cuda(data, "data")
    _require_cuda(digests, "digests")
    mc = cuts.numel() if max_cuts is None else int(max_cuts)
    rc = lib().seqcdc_fingerprint(data.data_ptr() if data.numel() else None, cuts.data_ptr() if mc else None,
                                  ncuts.data_ptr(), mc, digests.data_ptr() if mc else None,
                                  _stream_ptr(stream, data.device))
    _check(rc, "seqcdc_fingerprint")


def dedup_into(digests, cuts, ncuts, unique_bytes, first=None, max_cuts=None, workspace=None, stream=None) -> None:
    """Asynchronous seqcdc_dedup: first-occurrence flags (optional uint8 CUDA) and
    the stored bytes (int64 CUDA [1])."""
    _require_cuda(digests, "digests")
    mc = cuts.numel() if max_cuts is None else int(max_cuts)
    ws_ptr, ws_len = (workspace.data_ptr(), workspace.numel()) if workspace is not None else (None, 0)
    rc = lib().seqcdc_dedup(digests.data_ptr() if mc else None, cuts.data_ptr() if mc else None, ncuts.data_ptr(),
                            mc, first.data_ptr() if first is not None else None, unique_bytes.data_ptr(), ws_ptr,
                            ws_len, _stream_ptr(stream, digests.device))
    _check(rc, "seqcdc_dedup")


def dedup_workspace_size(max_cuts: int) -> int:
    return int(lib().seqcdc_dedup_workspace_size(int(max_cuts)))


def range_resync_dev_into(buf, range_len: int, d_entry, global_offset: int, p: SeqParams, spec, spec_n, cuts, ncuts,
                          status, stream=None) -> None:
    """Asynchronous seqcdc_range_resync_dev: the entry (a global offset) is read on
    the device from ``d_entry`` (an int64 CUDA tensor element), no host sync."""
    _require_cuda(buf, "buf")
    _require_out(cuts, "cuts", range_max_cuts(buf.numel(), range_len, p), buf)
    _require_out(status, "status", 4, buf)
    cp = p.c()
    rc = lib().seqcdc_range_resync_dev(buf.data_ptr() if buf.numel() else None, buf.numel(), range_len,
                                       d_entry.data_ptr(), global_offset, ctypes.byref(cp),
                                       spec.data_ptr() if spec.numel() else None, spec_n.data_ptr(),
                                       cuts.data_ptr() if cuts.numel() else None, ncuts.data_ptr(),
                                       status.data_ptr(), _stream_ptr(stream, buf.device))
    _check(rc, "seqcdc_range_resync_dev")


def range_chunk_tail_into(buf, range_len: int, global_offset: int, p: SeqParams, cuts, ncuts, tail_max: int,
                          block, workspace=None, stream=None) -> None:
    """Asynchronous seqcdc_range_chunk_tail (entry 0): the speculative chain of the
    range, and its exchange block (int64 CUDA [3 + tail_max] = overhang, count,
    tail_n, tail)."""
    _require_cuda(buf, "buf")
    _require_out(cuts, "cuts", range_max_cuts(buf.numel(), range_len, p), buf)
    _require_out(ncuts, "ncuts", 1, buf)
    _require_out(block, "block", 3 + tail_max, buf)
    cp = p.c()
    ws_ptr, ws_len = (workspace.data_ptr(), workspace.numel()) if workspace is not None else (None, 0)
    b0 = block.data_ptr()
    rc = lib().seqcdc_range_chunk_tail(buf.data_ptr() if buf.numel() else None, buf.numel(), range_len, 0,
                                       global_offset, ctypes.byref(cp), cuts.data_ptr() if cuts.numel() else None,
                                       ncuts.data_ptr(), tail_max, b0 + 24 if tail_max else None,
                                       b0 + 16 if tail_max else None, b0, ws_ptr, ws_len,
                                       _stream_ptr(stream, buf.device))
    _check(rc, "seqcdc_range_chunk_tail")


def range_merge_tail_into(buf, range_len: int, global_offset: int, p: SeqParams, prev_block, tail_max: int, spec,
                          spec_n, cuts, ncuts, status, spec_ov=None, sum3=None, stream=None) -> None:
    """Asynchronous seqcdc_range_merge_tail: ``prev_block`` = the previous range's
    exchange block; ``sum3`` (optional int64 CUDA [3]) = final overhang, count,
    ``spec_ov[0]``."""
    _require_cuda(buf, "buf")
    _require_out(prev_block, "prev_block", 3 + tail_max, buf)
    _require_out(cuts, "cuts", range_max_cuts(buf.numel(), range_len, p), buf)
    _require_out(ncuts, "ncuts", 1, buf)
    _require_out(status, "status", 4, buf)
    cp = p.c()
    rc = lib().seqcdc_range_merge_tail(buf.data_ptr() if buf.numel() else None, buf.numel(), range_len,
                                       global_offset, ctypes.byref(cp), prev_block.data_ptr(), tail_max,
                                       spec.data_ptr() if spec.numel() else None, spec_n.data_ptr(),
                                       cuts.data_ptr() if cuts.numel() else None, ncuts.data_ptr(),
                                       status.data_ptr(), spec_ov.data_ptr() if spec_ov is not None else None,
                                       sum3.data_ptr() if sum3 is not None else None, _stream_ptr(stream, buf.device))
    _check(rc, "seqcdc_range_merge_tail")


# ---------------------------------------------------------------- fused exchange over peer memory
IPC_HANDLE_BYTES = 64


def xchg_alloc(nbytes: int):
    """A zeroed device mailbox of ``nbytes`` owned by this process (free with
    xchg_free) and its CUDA IPC handle (bytes) for the other ranks."""
    ptr = ctypes.c_void_p()
    h = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
    _check(lib().seqcdc_xchg_alloc(int(nbytes), ctypes.byref(ptr), h), "seqcdc_xchg_alloc")
    return int(ptr.value), bytes(h.raw)


def xchg_open(handle: bytes) -> int:
    """Map another process's mailbox; returns its device address in this process."""
    if len(handle) != IPC_HANDLE_BYTES:
        raise SeqCDCError("IPC handle must be 64 bytes")
    ptr = ctypes.c_void_p()
    _check(lib().seqcdc_xchg_open(handle, ctypes.byref(ptr)), "seqcdc_xchg_open")
    return int(ptr.value)


def xchg_close(peer_ptr: int) -> None:
    _check(lib().seqcdc_xchg_close(peer_ptr), "seqcdc_xchg_close")


def xchg_free(ptr: int) -> None:
    _check(lib().seqcdc_xchg_free(ptr), "seqcdc_xchg_free")


def range_chunk_tail_push_into(buf, range_len: int, global_offset: int, p: SeqParams, cuts, ncuts, tail_max: int,
                               block, peer_blk: int, peer_flag: int, flag_value: int, workspace=None,
                               stream=None) -> None:
    """range_chunk_tail_into whose last kernel also stores the exchange block
    into a mapped peer mailbox (``peer_blk``, 3 + tail_max int64) and releases
    ``flag_value`` to ``peer_flag`` (device addresses from xchg_open)."""
    _require_cuda(buf, "buf")
    _require_out(cuts, "cuts", range_max_cuts(buf.numel(), range_len, p), buf)
    _require_out(ncuts, "ncuts", 1, buf)
    _require_out(block, "block", 3 + tail_max, buf)
    cp = p.c()
    ws_ptr, ws_len = (workspace.data_ptr(), workspace.numel()) if workspace is not None else (None, 0)
    b0 = block.data_ptr()
    rc = lib().seqcdc_range_chunk_tail_push(buf.data_ptr() if buf.numel() else None, buf.numel(), range_len, 0,
                                            global_offset, ctypes.byref(cp),
                                            cuts.data_ptr() if cuts.numel() else None, ncuts.data_ptr(), tail_max,
                                            b0 + 24 if tail_max else None, b0 + 16 if tail_max else None, b0,
                                            ws_ptr, ws_len, peer_blk, peer_flag, int(flag_value),
                                            _stream_ptr(stream, buf.device))
    _check(rc, "seqcdc_range_chunk_tail_push")


def range_merge_tail_wait_into(buf, range_len: int, global_offset: int, p: SeqParams, mailbox: int, flag: int,
                               flag_value: int, tail_max: int, spec, spec_n, cuts, ncuts, status, spec_ov=None,
                               sum3=None, timeout_ns: int = 2_000_000_000, stream=None) -> None:
    """range_merge_tail_into reading the previous range's block from this rank's
    mailbox (device address) once ``flag`` reaches ``flag_value`` (waited for on
    the device; a timeout reports overhang UINT64_MAX in ``sum3``)."""
    _require_cuda(buf, "buf")
    _require_out(cuts, "cuts", range_max_cuts(buf.numel(), range_len, p), buf)
    _require_out(ncuts, "ncuts", 1, buf)
    _require_out(status, "status", 4, buf)
    cp = p.c()
    rc = lib().seqcdc_range_merge_tail_wait(buf.data_ptr() if buf.numel() else None, buf.numel(), range_len,
                                            global_offset, ctypes.byref(cp), mailbox, tail_max,
                                            spec.data_ptr() if spec.numel() else None, spec_n.data_ptr(),
                                            cuts.data_ptr() if cuts.numel() else None, ncuts.data_ptr(),
                                            status.data_ptr(), spec_ov.data_ptr() if spec_ov is not None else None,
                                            sum3.data_ptr() if sum3 is not None else None, flag, int(flag_value),
                                            int(timeout_ns), _stream_ptr(stream, buf.device))
    _check(rc, "seqcdc_range_merge_tail_wait")


def xchg_put_rows_into(src, tables, row: int, step: int, stream=None) -> None:
    """Store ``src`` (int64 CUDA [nwords]) into row ``row`` of every rank's table
    (``tables``: int64 CUDA [nranks] of mapped table addresses) and release
    ``step`` behind it."""
    _require_cuda(src, "src")
    _check(lib().seqcdc_xchg_put_rows(src.data_ptr(), src.numel(), tables.data_ptr(), tables.numel(), row,
                                      int(step), _stream_ptr(stream, src.device)), "seqcdc_xchg_put_rows")


def xchg_wait_rows_into(table: int, nwords: int, nranks: int, step: int, status, out=None,
                        timeout_ns: int = 10_000_000_000, stream=None) -> None:
    """Wait on the device until all rows of this rank's table (device address)
    carry ``step``; the rows' data packed into ``out`` (int64 CUDA
    [nranks*nwords], optional); ``status`` (int64 CUDA [1]) = 0, or 1 on timeout."""
    _require_cuda(status, "status")
    _check(lib().seqcdc_xchg_wait_rows(table, nwords, nranks, int(step), int(timeout_ns), status.data_ptr(),
                                       out.data_ptr() if out is not None else None,
                                       _stream_ptr(stream, status.device)), "seqcdc_xchg_wait_rows")
