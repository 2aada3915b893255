"""GPU parity of the step after chunking (NEXT-1): per-chunk SHA-256 digests
(seqcdc_fingerprint) byte for byte against the oracle's hashlib digests, and
the dedup index (seqcdc_dedup) -- first-occurrence flags and stored bytes --
against the oracle's set-based definition (Eq. 1)."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2505_21194_b200 as sc  # noqa: E402


def _gpu_fp(b: np.ndarray, cuts: np.ndarray, offset: int = 0):
    buf = torch.zeros(b.size + offset + 64, dtype=torch.uint8, device="cuda")
    buf[offset:offset + b.size] = torch.from_numpy(b).cuda()
    d = buf[offset:offset + b.size]
    c = torch.from_numpy(cuts.astype(np.int64)).cuda()
    nc = torch.tensor([cuts.size], dtype=torch.int64, device="cuda")
    dg = torch.empty(max(cuts.size, 1) * 32, dtype=torch.uint8, device="cuda")
    sc.fingerprint_into(d, c, nc, dg, max_cuts=cuts.size)
    return dg[: 32 * cuts.size].cpu().numpy().reshape(-1, 32), c, nc, dg


def test_sha256_padding_edges_and_alignment():
    """Every chunk length 0..200 (all padding cases: rem <= 55, 56..63, multiples
    of 64) at every start alignment 0..15."""
    rng = np.random.default_rng(7)
    lens = np.array(list(range(0, 201)) + [1000, 4095, 4096, 4097, 8191])
    b = rng.integers(0, 256, int(lens.sum())).astype(np.uint8)
    cuts = np.cumsum(lens)
    for off in range(16):
        got, *_ = _gpu_fp(b, cuts, off)
        assert np.array_equal(got, oracle.fingerprints(b, cuts)), off


def test_fingerprints_of_chunked_stream():
    b = synth.fill_host("markov", 5, 0, 6 << 20)
    p = oracle.table1(4, 1)
    cuts = oracle.chunk(b, p)
    got, *_ = _gpu_fp(b, cuts, 3)
    assert np.array_equal(got, oracle.fingerprints(b, cuts))


def test_dedup_index_versions():
    """Scaled config 4 (versioned backups): chunk on the GPU, fingerprint and
    index on the GPU, no host sync in between; flags and stored bytes equal the
    oracle's."""
    d, _ = synth.versions_device(4, 8 << 20)
    b = d.cpu().numpy()
    p = oracle.table1(16)
    P = sc.SeqParams(p.mode, p.seq_length, p.skip_trigger, p.skip_size, p.min_size, p.max_size)
    mc = sc.max_cuts(d.numel(), P)
    cuts = torch.empty(mc, dtype=torch.int64, device="cuda")
    nc = torch.zeros(1, dtype=torch.int64, device="cuda")
    dg = torch.empty(32 * mc, dtype=torch.uint8, device="cuda")
    first = torch.zeros(mc, dtype=torch.uint8, device="cuda")
    uniq = torch.zeros(1, dtype=torch.int64, device="cuda")
    sc.chunk_into(d, P, cuts, nc)
    sc.fingerprint_into(d, cuts, nc, dg, max_cuts=mc)
    sc.dedup_into(dg, cuts, nc, uniq, first=first, max_cuts=mc)
    k = int(nc.item())
    want_cuts = oracle.chunk(b, p)
    assert np.array_equal(cuts[:k].cpu().numpy().astype(np.uint64), want_cuts)
    wfirst, wuniq = oracle.dedup(b, want_cuts)
    assert np.array_equal(first[:k].cpu().numpy().astype(bool), wfirst)
    assert int(uniq.item()) == wuniq
    assert 0.5 < wuniq / b.size < 0.7


def test_dedup_all_duplicates_and_empty():
    blk = np.random.default_rng(3).integers(0, 256, 5000).astype(np.uint8)
    b = np.tile(blk, 40)
    cuts = np.arange(5000, b.size + 1, 5000)
    got, c, nc, dg = _gpu_fp(b, cuts)
    uniq = torch.zeros(1, dtype=torch.int64, device="cuda")
    first = torch.zeros(cuts.size, dtype=torch.uint8, device="cuda")
    sc.dedup_into(dg, c, nc, uniq, first=first, max_cuts=cuts.size)
    assert int(uniq.item()) == 5000
    assert first.cpu().numpy().tolist() == [1] + [0] * 39
    z = torch.zeros(0, dtype=torch.int64, device="cuda")
    nz = torch.zeros(1, dtype=torch.int64, device="cuda")
    sc.dedup_into(dg, z, nz, uniq, max_cuts=0)
    assert int(uniq.item()) == 0
