"""Multi-GPU SeqCDC: one huge stream sharded into contiguous ranges, one rank per GPU
(BASELINE config 5).

Why it shards: "the next cut depends only on the previous cut" -- f(base)
reads only [base, f(base)) and the stream end (P:179 sub-minimum skip, P:189
content skip, P:266 max cut all restart from the chunk start).  So every rank
chunks its own range at once, speculatively, as if a chunk started at its range
start; only the seam needs fixing, and the fix is local once the previous
rank's overhang (its first cut >= this range's start) is known.

Protocol, per rank r of P (SPMD; ``torch.distributed``, NCCL on GPUs, gloo in
the CPU tests):

1. ``spec``: the chain from the range start R_r, up to its first cut >= R_{r+1}
   (the overhang O_r).  Rank 0's chain is the true one (the stream starts there).
2. all_gather (O_r, count_r).
3. Rank r > 0 re-synchronises from the true entry O_{r-1}: re-walk until a cut
   coincides with the speculative chain (then the rest is reused).  If the
   re-walk reaches R_{r+1} without merging (phase-locked data), rank r's
   overhang changes.
4. all_gather (O_r, count_r).  If every overhang equals the one its successor
   used, the result is final; otherwise the ranks whose entry changed repeat
   3-4 (at most P-1 rounds; normally one).
5. Exclusive prefix of the counts = each rank's first global cut index.

The cut lists stay sharded: rank r owns the chunks that START in [R_r, R_{r+1}),
i.e. cuts (O_{r-1}, O_r] -- concatenated over ranks they are exactly the
single-stream cut list.

The byte work is done by a backend; ``CudaRangeBackend`` drives the C-ABI range
calls (seqcdc_range_chunk / seqcdc_range_resync) and is the only product
backend.  The CPU tests plug in an oracle-based backend to check the protocol
itself with world_size > 1 over gloo.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Any

import torch
import torch.distributed as dist


@dataclass
class Shard:
    """Rank-local piece of a stream: ``buf`` = bytes [global_offset,
    global_offset + len(buf)): the range (first ``range_len`` bytes) plus a
    right halo of >= max_size - 1 bytes, or, for the last rank, exactly the
    rest of the stream.  ``stream_len`` (optional) lets a non-final range's
    halo be shorter when it reaches the end of the stream."""

    buf: Any
    range_len: int
    global_offset: int
    stream_len: int | None = None


@dataclass
class Chain:
    """A backend's cut list for one shard: ``count`` cuts (global offsets)
    ending at ``overhang`` (the first cut >= the range end, or the stream end)."""

    cuts: Any
    count: int
    overhang: int
    extra: dict = field(default_factory=dict)


@dataclass
class ShardResult:
    cuts: Any            # this rank's true cuts (global offsets): cuts[:count]
    count: int
    first_index: int     # global index of cuts[0] in the whole stream's list
    total: int           # number of cuts of the whole stream
    rounds: int          # exchange rounds after the speculative pass (1 normally)
    resync_cuts: int     # cuts re-walked by this rank
    entry: int           # global offset where this rank's first chunk starts


def _allgather_i64(values, group, device):
    t = torch.tensor(values, dtype=torch.int64, device=device)
    ws = dist.get_world_size(group)
    out = [torch.empty_like(t) for _ in range(ws)]
    dist.all_gather(out, t, group=group)
    return torch.stack(out).cpu().tolist()


def _allgather_dev(t, group):
    """all_gather of a small device tensor, stream-ordered (no host sync)."""
    P = dist.get_world_size(group)
    out = torch.empty((P,) + tuple(t.shape), dtype=t.dtype, device=t.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, t.contiguous(), group=group)
    else:
        dist.all_gather(list(out.unbind(0)), t.contiguous(), group=group)
    return out


def chunk_sharded(shard: Shard, backend, group=None, comm_device=None) -> ShardResult:
    """Run the sharded protocol for this rank (collective: every rank calls it).
    Backends with a device path (the CUDA one, exchanging over NCCL) enqueue the
    speculative pass, both exchanges and the re-synchronisation without a host
    sync and check once at the end (`_device_round`); the host loop below
    handles everything else, including further rounds when an overhang changed."""
    P = dist.get_world_size(group)
    r = dist.get_rank(group)
    dev = comm_device if comm_device is not None else backend.comm_device
    if P > 1 and r < P - 1:
        if shard.range_len < backend.max_size:
            raise ValueError("a non-final range must hold at least max_size bytes")
        # the chunk starting at the range's last true cut (< range end) reads up to
        # max_size - 1 bytes past the range end: without that right halo the
        # range call would treat the buffer end as the stream end and force a cut there
        at_end = shard.stream_len is not None and shard.global_offset + len(shard.buf) >= shard.stream_len
        if len(shard.buf) < shard.range_len + backend.max_size - 1 and not at_end:
            raise ValueError("a non-final range needs a right halo of >= max_size - 1 bytes "
                             f"(buffer {len(shard.buf)} < range {shard.range_len} + {backend.max_size - 1})")
    if getattr(backend, "device_protocol", False) and getattr(dev, "type", str(dev)) != "cpu":
        done = _device_round(shard, backend, group, P, r)
        if done is not None:
            backend.last_path = "p2p" if getattr(backend, "p2p", False) else "device"
            return done
    backend.last_path = "host"
    spec = backend.spec(shard)
    info = _allgather_i64([spec.overhang, spec.count], group, dev)
    return _host_rounds(shard, backend, group, dev, P, r, spec, info, spec, shard.global_offset, 0, 0)


def _device_round(shard, backend, group, P, r):
    """One exchange round, all enqueued on the stream; a single host read at the
    end decides whether it was final (the usual case) -- else None and the
    caller runs the host loop from scratch.

    Each rank's speculative pass also continues its chain ~96 cuts past its
    overhang (``tail``); one all_gather of (tail_n, overhang, tail) blocks lets
    rank r find where the true chain entering its range meets its own
    speculative chain -- a local search, no walking (seqcdc_range_merge_tail;
    a re-walk only if the tail is too short).  A second all_gather of
    (overhang, count, speculative overhang) gives the global prefix and proves
    no overhang changed."""
    if getattr(backend, "p2p", False):
        # fused exchange: rank r-1's last kernel stores its block straight into this
        # rank's mailbox over peer memory; the merge kernel waits for it on the device
        step = backend.next_step()
        spec = backend.spec_dev_tail(shard, last=(r == P - 1), push_step=step)
        cur = backend.merge_dev_wait(shard, spec, step) if r > 0 else spec
    else:
        spec = backend.spec_dev_tail(shard, last=(r == P - 1))   # extra: "block" [3 + E]
        blocks = _allgather_dev(spec.extra["block"], group)     # [P, 3 + E]
        cur = backend.merge_dev(shard, blocks[r - 1], spec) if r > 0 else spec
    s3 = cur.extra["sum3"] if r > 0 else spec.extra["block"][[0, 1, 0]]   # rank 0's chain is final
    if getattr(backend, "p2p", False):                      # rows stored into every rank's table, one host read
        h = backend.exchange_rows(s3, step)
    else:
        info = _allgather_dev(s3, group)                    # [P, 3] = final ov, count, speculative ov
        h = info.reshape(-1).cpu().tolist()
    if any(h[3 * k] != h[3 * k + 2] for k in range(P)):     # an overhang changed: more rounds needed
        return None
    counts = [h[3 * k + 1] for k in range(P)]
    entry = h[3 * (r - 1)] if r > 0 else shard.global_offset
    return ShardResult(cur.cuts, counts[r], sum(counts[:r]), sum(counts), 1, 0, entry)


def _host_rounds(shard, backend, group, dev, P, r, spec, info, cur, cur_entry, rounds, rewalked):
    while True:
        true_entry = info[r - 1][0] if r > 0 else shard.global_offset
        changed = 0
        if true_entry != cur_entry:
            cur = backend.resync(shard, true_entry - shard.global_offset, spec)
            rewalked = cur.extra.get("rewalked", 0)
            cur_entry, changed = true_entry, 1
        new = _allgather_i64([cur.overhang, cur.count, changed], group, dev)
        rounds += 1
        stable = all(new[k][0] == info[k][0] for k in range(P))
        info = new
        if stable:
            break
        if rounds > P + 1:
            raise RuntimeError("seam re-synchronisation did not converge")
    counts = [row[1] for row in info]
    return ShardResult(cur.cuts, cur.count, sum(counts[:r]), sum(counts), rounds, rewalked, cur_entry)


class CudaRangeBackend:
    """The product backend: the C-ABI range calls on the rank's GPU.  Buffers
    are allocated once per shard size and reused across calls."""

    TAIL = 96          # cuts each range continues past its overhang (device protocol)

    def __init__(self, params, device=None, stream=None):
        from . import SeqParams  # noqa: F401  (type of params)
        self.p = params
        self.max_size = params.max_size
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.comm_device = self.device
        self.stream = stream
        self.device_protocol = True      # spec_dev / resync_dev: no host sync inside a round
        self._key = None
        self.p2p = False                 # fused exchange over peer memory (enable_p2p)
        self._mb = self._peer = None
        self._peers = {}
        self._step = 0

    # ---- fused exchange over peer memory (SURVEY.md 8(e) "fused alternative")
    def enable_p2p(self, group=None) -> bool:
        """Give this rank a device mailbox (CUDA IPC) and map every other rank's,
        so that both exchanges of a step travel by peer stores (NVLink between
        GPUs) with device-side flags: rank r's last kernel stores its tail block
        into rank r+1's mailbox, and each rank stores its (overhang, count,
        speculative overhang) row into every rank's table -- no collective and
        no host involvement until the one host read of the table.  Collective:
        every rank calls it once; it is on only if every rank mapped every peer."""
        from . import xchg_alloc, xchg_open
        P, r = dist.get_world_size(group), dist.get_rank(group)
        if P < 2:
            return False
        self._P, self._r = P, r
        self._flag_off = ((8 * (3 + self.TAIL) + 127) // 128) * 128
        self._tab_off = self._flag_off + 128                 # two tables (step parity) of P rows x 4 words
        nbytes = self._tab_off + 2 * P * 32
        err, h = "", b""
        try:                             # any failure is reported to every rank below
            with torch.cuda.device(self.device):
                self._mb, h = xchg_alloc(nbytes)
        except Exception as e:           # noqa: BLE001
            err = f"alloc: {e}"
        handles = [None] * P
        dist.all_gather_object(handles, h, group=group)
        bases = [0] * P
        if not err:
            bases[r] = self._mb
            try:
                with torch.cuda.device(self.device):
                    for q in range(P):
                        if q != r:
                            if not handles[q]:
                                raise RuntimeError(f"rank {q} has no mailbox")
                            self._peers[q] = xchg_open(handles[q])
                            bases[q] = self._peers[q]
            except Exception as e:       # noqa: BLE001
                err = f"open: {e}"
        # every rank must agree, or the ranks would run different exchanges
        errs = [None] * P
        dist.all_gather_object(errs, err, group=group)
        self._step = 0
        self.p2p = not any(errs)
        if not self.p2p:
            self.close()
            self.p2p_error = next(e for e in errs if e)
            return False
        self._peer = bases[r + 1] if r + 1 < P else None
        # per step parity: the device array of every rank's table, and this rank's own
        self._tables = [torch.tensor([b + self._tab_off + k * P * 32 for b in bases], dtype=torch.int64,
                                     device=self.device) for k in range(2)]
        self._tabdev = torch.zeros(P * 3 + 1, dtype=torch.int64, device=self.device)   # rows, then status
        self._tabhost = torch.empty(P * 3 + 1, dtype=torch.int64, pin_memory=True)
        return True

    def exchange_rows(self, sum3, step: int, timeout_ns: int = 10_000_000_000) -> list[int]:
        """The step's second exchange over peer memory: store this rank's row
        (final overhang, count, speculative overhang) into every rank's table,
        wait for all rows of this step on the device, then one host read.
        Returns the P x 3 values row-major (raises after the timeout)."""
        from . import xchg_put_rows_into, xchg_wait_rows_into
        P, k = self._P, step & 1
        with torch.cuda.device(self.device):
            xchg_put_rows_into(sum3.contiguous(), self._tables[k], self._r, step, stream=self.stream)
            own = self._mb + self._tab_off + k * P * 32
            xchg_wait_rows_into(own, 3, P, step, self._tabdev[P * 3:], out=self._tabdev[: P * 3],
                                timeout_ns=timeout_ns, stream=self.stream)
            st = self.stream if self.stream is not None else torch.cuda.current_stream(self.device)
            with torch.cuda.stream(st):
                self._tabhost.copy_(self._tabdev, non_blocking=True)
            st.synchronize()
        h = self._tabhost.tolist()
        if h[P * 3] != 0:
            raise RuntimeError("peer-memory exchange timed out (a rank stopped responding)")
        return h[: P * 3]

    def next_step(self) -> int:
        self._step += 1
        return self._step

    def close(self) -> None:
        """Unmap the peer mailboxes and free this rank's (after all ranks are done)."""
        from . import xchg_close, xchg_free
        for q in list(self._peers):
            xchg_close(self._peers.pop(q))
        self._peer = None
        if self._mb is not None:
            xchg_free(self._mb)
            self._mb = None
        self.p2p = False

    def _alloc(self, shard: Shard):
        from . import range_max_cuts, workspace_size
        key = (shard.buf.numel(), shard.range_len)
        if key == self._key:
            return
        n, rl = key
        cap = max(range_max_cuts(n, rl, self.p), 1)
        dev = self.device
        self.spec_cuts = torch.empty(cap, dtype=torch.int64, device=dev)
        self.out_cuts = torch.empty(cap, dtype=torch.int64, device=dev)
        self.spec_n = torch.zeros(1, dtype=torch.int64, device=dev)
        self.out_n = torch.zeros(1, dtype=torch.int64, device=dev)
        self.status = torch.zeros(4, dtype=torch.int64, device=dev)
        self.ws = torch.empty(workspace_size(n, 1, self.p), dtype=torch.uint8, device=dev)
        self.host = torch.empty(8, dtype=torch.int64, pin_memory=True)
        self.block = torch.zeros(3 + self.TAIL, dtype=torch.int64, device=dev)   # ov, count, tail_n, tail
        self.sum3 = torch.zeros(3, dtype=torch.int64, device=dev)
        self._key = key

    def _read(self, cuts, ncuts, extra=None) -> list[int]:
        # one small D2H: count, last cut (the overhang) and the status words
        k = ncuts.clone()
        parts = [k, cuts[(k - 1).clamp_min(0)]] + ([extra] if extra is not None else [])
        with torch.cuda.stream(self.stream) if self.stream is not None else torch.cuda.device(self.device):
            v = torch.cat(parts)
            self.host[: v.numel()].copy_(v, non_blocking=True)
        (self.stream or torch.cuda.current_stream(self.device)).synchronize()
        return [int(x) for x in self.host[: v.numel()].tolist()]

    def spec(self, shard: Shard) -> Chain:
        from . import range_chunk_into
        self._alloc(shard)
        range_chunk_into(shard.buf, shard.range_len, 0, shard.global_offset, self.p, self.spec_cuts, self.spec_n,
                         workspace=self.ws, stream=self.stream)
        k, last = self._read(self.spec_cuts, self.spec_n)
        if k == 0:
            last = shard.global_offset
        return Chain(self.spec_cuts, k, last)

    def resync(self, shard: Shard, entry: int, spec: Chain) -> Chain:
        from . import range_resync_into
        self._alloc(shard)
        range_resync_into(shard.buf, shard.range_len, entry, shard.global_offset, self.p, spec.cuts, self.spec_n,
                          self.out_cuts, self.out_n, self.status, stream=self.stream)
        k, last, *st = self._read(self.out_cuts, self.out_n, self.status)
        if k == 0:
            last = shard.global_offset + entry
        return Chain(self.out_cuts, k, last, {"merged": bool(st[0]), "rewalked": int(st[1])})

    # ---- device path: summaries stay on the GPU (for NCCL all_gather), no host sync
    def _summary(self, cuts, ncuts, empty_overhang: int):
        k = ncuts.reshape(1)
        last = cuts.gather(0, (k - 1).clamp_min(0))
        ov = torch.where(k > 0, last, torch.full_like(last, empty_overhang))
        return torch.cat([ov, k])

    def spec_dev(self, shard: Shard) -> Chain:
        from . import range_chunk_into
        self._alloc(shard)
        with torch.cuda.device(self.device):
            range_chunk_into(shard.buf, shard.range_len, 0, shard.global_offset, self.p, self.spec_cuts, self.spec_n,
                             workspace=self.ws, stream=self.stream)
            sm = self._summary(self.spec_cuts, self.spec_n, shard.global_offset)
        return Chain(self.spec_cuts, -1, -1, {"sum": sm})

    def resync_dev(self, shard: Shard, d_entry, spec: Chain) -> Chain:
        """d_entry: int64 CUDA tensor [1] holding the true entry as a global offset."""
        from . import range_resync_dev_into
        self._alloc(shard)
        with torch.cuda.device(self.device):
            e = d_entry.contiguous()
            range_resync_dev_into(shard.buf, shard.range_len, e, shard.global_offset, self.p, spec.cuts,
                                  self.spec_n, self.out_cuts, self.out_n, self.status, stream=self.stream)
            sm = torch.cat([self.status[3:4], self.out_n.reshape(1)])
        return Chain(self.out_cuts, -1, -1, {"sum": sm})

    # ---- one-exchange device protocol (tails)
    def spec_dev_tail(self, shard: Shard, last: bool, push_step: int = 0) -> Chain:
        from . import range_chunk_tail_into, range_chunk_tail_push_into
        self._alloc(shard)
        E = 0 if last else self.TAIL
        with torch.cuda.device(self.device):
            if last:
                self.block[2].zero_()
            if push_step and not last:
                range_chunk_tail_push_into(shard.buf, shard.range_len, shard.global_offset, self.p, self.spec_cuts,
                                           self.spec_n, E, self.block, self._peer, self._peer + self._flag_off,
                                           push_step, workspace=self.ws, stream=self.stream)
            else:
                range_chunk_tail_into(shard.buf, shard.range_len, shard.global_offset, self.p, self.spec_cuts,
                                      self.spec_n, E, self.block, workspace=self.ws, stream=self.stream)
        # exchange block = (overhang, count, tail_n, tail); the second exchange
        # for rank 0 is (overhang, count, overhang): its chain is final already
        return Chain(self.spec_cuts, -1, -1, {"block": self.block})

    def merge_dev(self, shard: Shard, prev_block, spec: Chain) -> Chain:
        from . import range_merge_tail_into
        self._alloc(shard)
        with torch.cuda.device(self.device):
            pb = prev_block.contiguous()
            range_merge_tail_into(shard.buf, shard.range_len, shard.global_offset, self.p, pb, self.TAIL, spec.cuts,
                                  self.spec_n, self.out_cuts, self.out_n, self.status, spec_ov=self.block,
                                  sum3=self.sum3, stream=self.stream)
        return Chain(self.out_cuts, -1, -1, {"sum3": self.sum3})

    def merge_dev_wait(self, shard: Shard, spec: Chain, step: int, timeout_ns: int = 2_000_000_000) -> Chain:
        from . import range_merge_tail_wait_into
        self._alloc(shard)
        with torch.cuda.device(self.device):
            range_merge_tail_wait_into(shard.buf, shard.range_len, shard.global_offset, self.p, self._mb,
                                       self._mb + self._flag_off, step, self.TAIL, spec.cuts, self.spec_n,
                                       self.out_cuts, self.out_n, self.status, spec_ov=self.block, sum3=self.sum3,
                                       timeout_ns=timeout_ns, stream=self.stream)
        return Chain(self.out_cuts, -1, -1, {"sum3": self.sum3})


# ---------------------------------------------------------------- batches of independent streams
def lpt_assign(sizes, P: int):
    """Longest-processing-time-first assignment of whole streams to P ranks
    ("assign whole streams to GPUs with LPT by size"): streams
    in decreasing size, each to the currently lightest rank (ties -> lowest
    rank).  Deterministic; returns a list of stream-index lists (ascending)."""
    import heapq
    order = sorted(range(len(sizes)), key=lambda j: (-int(sizes[j]), j))
    heap = [(0, r) for r in range(P)]
    out = [[] for _ in range(P)]
    for j in order:
        load, r = heapq.heappop(heap)
        out[r].append(j)
        heapq.heappush(heap, (load + int(sizes[j]), r))
    return [sorted(x) for x in out]


def chunk_batch_sharded(streams, p, group=None, device=None):
    """Chunk this rank's share of a batch of independent streams ("files are
    chunked independently"): no data-path collective, one all_reduce of
    the cut totals.  ``streams`` = {stream index: uint8 CUDA tensor} for the
    streams lpt_assign gave this rank.  Returns ({index: cuts (local offsets)},
    total cuts over all ranks)."""
    from . import chunk_batch
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    idx = sorted(streams)
    out = {}
    local = 0
    if idx:
        sizes = [streams[j].numel() for j in idx]
        offs = torch.zeros(len(idx) + 1, dtype=torch.int64)
        offs[1:] = torch.cumsum(torch.tensor(sizes, dtype=torch.int64), 0)
        data = torch.cat([streams[j].reshape(-1) for j in idx]).to(dev)
        cuts, ci = chunk_batch(data, offs.to(dev), p)
        ci = ci.cpu().tolist()
        offl = offs.tolist()
        for t, j in enumerate(idx):
            out[j] = cuts[ci[t]:ci[t + 1]] - offl[t]
        local = int(ci[-1])
    tot = torch.tensor([local], dtype=torch.int64, device=dev if dist.get_backend(group) == "nccl" else "cpu")
    dist.all_reduce(tot, group=group)
    return out, int(tot.item())
