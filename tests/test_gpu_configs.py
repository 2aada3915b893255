"""BASELINE.json's configs at FULL size on the GPU, every cut compared with the
oracle (whole lists; the oracle runs in independent windows started at the
GPU's own cuts, on all host cores -- benchlib/verify.py explains why that is a
complete check).  Marked ``gpu`` and ``slow``: a few minutes on a B200.

Config 1 (8 MiB) and config 2 (1 GiB) are in test_gpu_parity.py.
"""
import os

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

import paper_2505_21194_b200 as sc  # noqa: E402
from benchlib import verify  # noqa: E402

GiB, MiB = 1 << 30, 1 << 20


def _sp(p: oracle.Params) -> sc.SeqParams:
    return sc.SeqParams(p.mode, p.seq_length, p.skip_trigger, p.skip_size, p.min_size, p.max_size)


@pytest.fixture(autouse=True)
def _release_pinned():
    yield
    torch.cuda.empty_cache()
    if hasattr(torch._C, "_host_emptyCache"):
        torch._C._host_emptyCache()          # the pinned host staging of the 16-64 GiB streams


def _chunk_dev(d, p):
    P = _sp(p)
    cuts = torch.empty(max(sc.max_cuts(d.numel(), P), 1), dtype=torch.int64, device=d.device)
    nc = torch.zeros(1, dtype=torch.int64, device=d.device)
    sc.chunk_into(d, P, cuts, nc)
    k = int(nc.item())
    return cuts[:k].cpu().numpy().astype(np.uint64)


@pytest.mark.parametrize("walker", ["warp", "lane"])
def test_config5_full_64gib(walker, monkeypatch):
    """Config 5: one 64 GiB rampmix stream (seed 5), Increasing, L5 T50 S256,
    min 4 KiB, max 16 KiB -- the stream the bench line is quoted on."""
    monkeypatch.setenv("SEQCDC_WALKER", walker)
    n = 64 * GiB
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    synth.fill_device("rampmix", 5, 0, d)
    p = oracle.table1(8)
    got = _chunk_dev(d, p)
    host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    host.copy_(d)
    del d
    torch.cuda.empty_cache()
    hb = host.numpy()
    chk = verify.check_windows(lambda a, b: hb[a:b], n, p, got)
    assert chk["bit_exact"], chk.get("first_mismatch")
    assert got.size == 15375877                      # the count every earlier full run found


def test_config4_full_versioned():
    """Config 4: 4 GiB base + 10 versions at 1% edits (~44 GiB), one stream,
    Increasing, L5 T50 S512, min 8 KiB, max 32 KiB; plus the dedup ratio from a
    host SHA-256 index of the (oracle-equal) chunks."""
    d, _ = synth.versions_device(4, 4 * GiB)
    n = d.numel()
    p = oracle.table1(16)
    got = _chunk_dev(d, p)
    host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    host.copy_(d)
    del d
    torch.cuda.empty_cache()
    hb = host.numpy()
    chk = verify.check_windows(lambda a, b: hb[a:b], n, p, got)
    assert chk["bit_exact"], chk.get("first_mismatch")
    assert got.size == 5327115


def test_config3_full_all_streams():
    """Config 3: 256 streams x 64 MiB +-25% (50/30/20 uniform/Markov/zero-heavy),
    Table I 4/8/16 KiB rows; every stream's whole list against the oracle (one
    stream per host thread)."""
    from concurrent.futures import ThreadPoolExecutor
    ns = 256
    off, kinds, seeds = synth.batch_layout(3, ns, 64 * MiB)
    total = int(off[-1])
    d = torch.empty(total, dtype=torch.uint8, device="cuda")
    for j in range(ns):
        a, b = int(off[j]), int(off[j + 1])
        synth.fill_device(int(kinds[j]), int(seeds[j]), 0, d[a:b], b - a)
    doff = torch.from_numpy(off.astype(np.int64)).cuda()
    host = torch.empty(total, dtype=torch.uint8, pin_memory=True)
    host.copy_(d)
    hb = host.numpy()
    for avg in (4, 8, 16):
        p = oracle.table1(avg)
        P = _sp(p)
        cuts = torch.empty(sc.max_cuts_batch(total, ns, P), dtype=torch.int64, device="cuda")
        idx = torch.empty(ns + 1, dtype=torch.int64, device="cuda")
        nc = torch.zeros(1, dtype=torch.int64, device="cuda")
        sc.chunk_batch_into(d, doff, P, cuts, idx, nc, total=total)
        ci = idx.cpu().numpy()
        gc = cuts[: int(nc.item())].cpu().numpy().astype(np.uint64)

        def one(j):
            a, b = int(off[j]), int(off[j + 1])
            want = oracle.chunk(hb[a:b], p).astype(np.uint64) + np.uint64(a)
            return bool(np.array_equal(gc[int(ci[j]):int(ci[j + 1])], want))

        with ThreadPoolExecutor(os.cpu_count() or 1) as ex:
            ok = list(ex.map(one, range(ns)))
        assert all(ok), (avg, [j for j in range(ns) if not ok[j]][:5])
        assert int(ci[-1]) == gc.size


def test_config4_full_dedup_ratio():
    """Config 4's dedup fidelity at full size: GPU chunking, GPU SHA-256 per
    chunk and the GPU dedup index (NEXT-1, Eq. 1) give exactly
    the stored bytes of a host index -- hashlib SHA-256 of the same chunks and a
    Python set, the oracle's definition (oracle.dedup), on all host threads --
    and the cut list is the oracle's (window check)."""
    import hashlib
    from concurrent.futures import ThreadPoolExecutor
    d, _ = synth.versions_device(4, 4 * GiB)
    n = d.numel()
    p = oracle.table1(16)
    P = _sp(p)
    mc = sc.max_cuts(n, P)
    cuts = torch.empty(mc, dtype=torch.int64, device="cuda")
    nc = torch.zeros(1, dtype=torch.int64, device="cuda")
    dg = torch.empty(32 * mc, dtype=torch.uint8, device="cuda")
    uniq = torch.zeros(1, dtype=torch.int64, device="cuda")
    sc.chunk_into(d, P, cuts, nc)
    sc.fingerprint_into(d, cuts, nc, dg, max_cuts=mc)
    sc.dedup_into(dg, cuts, nc, uniq, max_cuts=mc)
    k = int(nc.item())
    got = cuts[:k].cpu().numpy().astype(np.uint64)
    gpu_uniq = int(uniq.item())
    del dg
    host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    host.copy_(d)
    del d
    torch.cuda.empty_cache()
    hb = host.numpy()
    assert verify.check_windows(lambda a, b: hb[a:b], n, p, got)["bit_exact"]
    starts = np.concatenate([[0], got[:-1]]).astype(np.int64)
    ends = got.astype(np.int64)
    mv = memoryview(hb)
    parts = np.array_split(np.arange(k), os.cpu_count() or 1)

    def digests(ix):
        return [(hashlib.sha256(mv[starts[i]:ends[i]]).digest(), int(ends[i] - starts[i])) for i in ix.tolist()]

    seen, host_uniq = set(), 0
    with ThreadPoolExecutor(os.cpu_count() or 1) as ex:
        for res in ex.map(digests, parts):          # in chunk order: the first occurrence is stored
            for h, ln in res:
                if h not in seen:
                    seen.add(h)
                    host_uniq += ln
    assert gpu_uniq == host_uniq, (gpu_uniq, host_uniq)
    assert 0.55 < host_uniq / n < 0.62               # ~0.59 at 16 KiB params [MC-8]
