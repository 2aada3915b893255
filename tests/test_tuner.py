"""NEXT-3 Monte-Carlo parameter search: its statistics on the CPU against a
direct computation, and on the GPU (batch kernel) against the oracle's cut
lists for the same streams."""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2505_21194_b200 import tuner


def _batch(ns=6, size=300_000, seed=9):
    streams = [synth.fill_host("uniform", seed + j, 0, size + 17 * j) for j in range(ns)]
    off = np.zeros(ns + 1, np.int64)
    off[1:] = np.cumsum([s.size for s in streams])
    return np.concatenate(streams), off


def test_chunk_stats_definition():
    b, off = _batch()
    p = oracle.table1(8)
    cuts, idx = oracle.chunk_batch(b, off, p)
    m, med, k, forced = tuner.chunk_stats(torch.from_numpy(cuts.astype(np.int64)), torch.from_numpy(idx.astype(np.int64)),
                                          torch.from_numpy(off), p.max_size)
    sizes = []
    for j in range(off.size - 1):
        c = cuts[idx[j]:idx[j + 1]].astype(np.int64)
        st = np.concatenate([[off[j]], c[:-1]])
        sizes += (c - st)[:-1].tolist()                   # drop the stream's final chunk
    assert k == len(sizes)
    assert m == pytest.approx(np.mean(sizes)) and med == pytest.approx(np.median(sizes))
    assert forced == pytest.approx(np.mean(np.asarray(sizes) == p.max_size))


def test_candidates_order():
    pts = [tuner.SweepPoint(5, t, 256, 2048, 8192, m, m, 10, 0.0) for t, m in [(40, 3900), (50, 4100), (60, 4600)]]
    c = tuner.candidates(pts, 4096, 0.05)
    assert [x.skip_trigger for x in c] == [50, 40]


@pytest.mark.gpu
def test_sweep_gpu_matches_oracle():
    b, off = _batch()
    d = torch.from_numpy(b).cuda()
    doff = torch.from_numpy(off).cuda()
    grid = [(5, 50, 256), (6, 40, 128), (4, 70, 512)]
    pts = tuner.sweep(d, doff, grid, 8)
    for pt in pts:
        p = oracle.Params(0, pt.seq_length, pt.skip_trigger, pt.skip_size, pt.min_size, pt.max_size)
        cuts, idx = oracle.chunk_batch(b, off, p)
        m, med, k, f = tuner.chunk_stats(torch.from_numpy(cuts.astype(np.int64)), torch.from_numpy(idx.astype(np.int64)),
                                         torch.from_numpy(off), p.max_size)
        assert (pt.median_chunk, pt.chunks) == (med, k)
        assert pt.mean_chunk == pytest.approx(m, rel=1e-12)   # device vs host summation order
