"""Config 4 (versioned backup stream, dedup fidelity), scaled: the seeded
version generator, and the dedup ratio (unique/total bytes under a SHA-256
chunk index, Eq. 1) computed from cut lists.  The GPU test
checks the CUDA cut list and its dedup ratio against the oracle's."""
import hashlib

import numpy as np
import pytest

import oracle
import synth

BASE = 16 << 20


def dedup_ratio(b: np.ndarray, cuts) -> float:
    """unique bytes / total bytes over the chunks cut at `cuts` (SHA-256 index)."""
    cuts = np.asarray(cuts, dtype=np.int64)
    starts = np.concatenate([[0], cuts[:-1]])
    seen, uniq = set(), 0
    mv = memoryview(b)
    for s, e in zip(starts.tolist(), cuts.tolist()):
        h = hashlib.sha256(mv[s:e]).digest()
        if h not in seen:
            seen.add(h)
            uniq += e - s
    return uniq / b.size


def test_version_edits_budget_and_disjoint():
    rng = np.random.default_rng([4, 4, 0])
    size = 1 << 22
    ed = synth._version_edits(rng, size, 0.01)
    assert sum(ln for _, ln, _ in ed) >= 0.01 * size
    prev_end = -1
    for pos, ln, op in ed:
        assert 1 <= ln <= 4096 and op in (0, 1, 2) and 0 <= pos
        end = pos if op == 0 else pos + ln
        assert end <= size and pos >= prev_end and (op != 0 or pos > prev_end or prev_end == -1 or pos >= prev_end)
        prev_end = max(prev_end, end)


def test_versions_host_deterministic_and_sized():
    b1, s1 = synth.versions_host(4, 1 << 20, nver=3)
    b2, s2 = synth.versions_host(4, 1 << 20, nver=3)
    assert s1 == s2 and np.array_equal(b1, b2) and b1.size == sum(s1)
    assert np.array_equal(b1[: 1 << 20], synth.fill_host("uniform", 4, 0, 1 << 20))
    # each version is mostly a copy of the previous one (1% edited)
    v0, v1 = b1[: s1[0]], b1[s1[0]: s1[0] + s1[1]]
    assert abs(s1[1] - s1[0]) < 0.02 * s1[0]
    assert np.mean(v0[:4096] == v1[:4096]) > 0.5 or np.mean(v0[-4096:] == v1[-4096:]) > 0.5


def test_dedup_ratio_statistics():
    """Sanity (not parity): SURVEY.md [MC-8] measured unique/total ~0.59 at the
    16 KiB Table I row and ~0.34 at 8 KiB on this stream shape; fixed-size 8 KiB
    chunking finds almost nothing (~1.0: every edit shifts all later blocks)."""
    b, _ = synth.versions_host(4, BASE)
    r16 = dedup_ratio(b, oracle.chunk(b, oracle.table1(16)))
    r8 = dedup_ratio(b, oracle.chunk(b, oracle.table1(8)))
    fixed = dedup_ratio(b, np.minimum(np.arange(8192, b.size + 8192, 8192), b.size))
    assert 0.50 < r16 < 0.70, r16
    assert 0.25 < r8 < 0.45, r8
    assert fixed > 0.95, fixed


@pytest.mark.gpu
def test_config4_scaled_gpu_parity_and_dedup():
    torch = pytest.importorskip("torch")
    import paper_2505_21194_b200 as sc
    d, sizes = synth.versions_device(4, BASE)
    b, sizes_h = synth.versions_host(4, BASE)
    assert sizes == sizes_h
    assert np.array_equal(d.cpu().numpy(), b)
    p = oracle.table1(16)
    got = sc.chunk(d, sc.SeqParams(p.mode, p.seq_length, p.skip_trigger, p.skip_size, p.min_size,
                                   p.max_size)).cpu().numpy().astype(np.uint64)
    want = oracle.chunk(b, p)
    assert np.array_equal(got, want)
    assert dedup_ratio(b, got) == dedup_ratio(b, want)
