"""Monte-Carlo parameter search (§5):
"to obtain the parameter value combination needed to generate a given average
chunk size, we first used Monte-Carlo simulations on randomized data streams ...
to identify candidate combinations resulting in an average chunk size of
4 KB" -- then the best one was picked on a real dataset (Table I).

Here every grid point is one ``seqcdc_chunk_batch`` call over a batch of
seeded random streams resident on the GPU (the batch kernel is the workload);
the per-stream final (partial) chunks are excluded from the statistics.  Under
this build's reading of SeqLength (bytes, DESIGN.md c1) Table I's rows give
means of about 0.55x their labels on random data; the search finds the rows
that hit the labels."""
from __future__ import annotations

from dataclasses import dataclass

import torch


@dataclass
class SweepPoint:
    seq_length: int
    skip_trigger: int
    skip_size: int
    min_size: int
    max_size: int
    mean_chunk: float
    median_chunk: float
    chunks: int
    forced_frac: float      # share of chunks that end at min(base + max, end): max-forced


def chunk_stats(cuts, cut_index, offsets, max_size: int):
    """Mean / median chunk size over complete chunks (each stream's last chunk
    excluded), from a batch cut list (device or host tensors)."""
    cuts = cuts.to(torch.int64)
    ci = cut_index.to(torch.int64)
    off = offsets.to(torch.int64)
    ns = off.numel() - 1
    # chunk starts: the previous cut, or the stream start for a stream's first chunk
    starts = torch.empty_like(cuts)
    starts[1:] = cuts[:-1]
    firsts = ci[:-1]
    nonempty = ci[1:] > ci[:-1]
    starts[firsts[nonempty]] = off[:-1][nonempty]
    sizes = cuts - starts
    keep = torch.ones_like(sizes, dtype=torch.bool)
    keep[(ci[1:] - 1)[nonempty]] = False                # each stream's final chunk
    s = sizes[keep]
    if s.numel() == 0:
        return 0.0, 0.0, 0, 0.0
    forced = (s == max_size).double().mean().item()
    return s.double().mean().item(), s.double().median().item(), int(s.numel()), forced


def sweep(data, offsets, grid, avg_kib: int, mode: int = 0, chunk_batch=None):
    """Run every (L, T, S) of ``grid`` with min = avg/2, max = 2*avg on the
    batch (``data`` uint8, ``offsets`` int64 [ns+1], same device)."""
    from . import SeqParams
    if chunk_batch is None:
        from . import chunk_batch
    avg = avg_kib * 1024
    out = []
    for L, T, S in grid:
        p = SeqParams(mode, L, T, S, avg // 2, 2 * avg)
        cuts, idx = chunk_batch(data, offsets, p)
        m, med, k, f = chunk_stats(cuts, idx, offsets, p.max_size)
        out.append(SweepPoint(L, T, S, p.min_size, p.max_size, m, med, k, f))
    return out


def candidates(points, target: float, tol: float = 0.05):
    """Grid points whose mean chunk is within tol of the target, closest first."""
    c = [p for p in points if abs(p.mean_chunk - target) <= tol * target]
    return sorted(c, key=lambda p: abs(p.mean_chunk - target))
