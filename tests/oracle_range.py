"""Oracle-based range backend for the CPU tests of the multi-GPU protocol
(paper_2505_21194_b200/dist.py).  TEST INFRASTRUCTURE: it computes each
rank's chains with the CPU oracle's f(base) (oracle.next_cut), so the gloo
tests check the exchange protocol itself, independent of the CUDA path."""
from __future__ import annotations

import numpy as np
import torch

import oracle
from paper_2505_21194_b200.dist import Chain, Shard


class OracleRangeBackend:
    comm_device = torch.device("cpu")

    def __init__(self, p: oracle.Params):
        self.p = p
        self.max_size = p.max_size

    def _walk(self, shard: Shard, start: int, stop_set=None):
        """Chain from local `start`: cuts until the first one >= range_len (or a
        cut in stop_set).  len(buf) is the stream end, as in the C ABI."""
        cuts, base, hit = [], start, None
        while base < shard.range_len:
            c = oracle.next_cut(shard.buf, base, self.p)
            g = shard.global_offset + c
            cuts.append(g)
            if stop_set is not None and g in stop_set:
                hit = g
                break
            base = c
        return cuts, hit

    def spec(self, shard: Shard) -> Chain:
        cuts, _ = self._walk(shard, 0)
        arr = np.asarray(cuts, dtype=np.uint64)
        return Chain(arr, arr.size, int(arr[-1]) if arr.size else shard.global_offset)

    def resync(self, shard: Shard, entry: int, spec: Chain) -> Chain:
        pos = {int(c): i for i, c in enumerate(spec.cuts)}
        cuts, hit = self._walk(shard, entry, pos)
        m = len(cuts)
        if hit is not None:
            cuts = cuts + [int(c) for c in spec.cuts[pos[hit] + 1:]]
        arr = np.asarray(cuts, dtype=np.uint64)
        ov = int(arr[-1]) if arr.size else shard.global_offset + entry
        return Chain(arr, arr.size, ov, {"merged": hit is not None, "rewalked": m})
