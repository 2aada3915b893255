"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle,
element by element, on seeded inputs.  Integer output => bit-exact.

Marked ``gpu``; run with ``pytest -m gpu`` on a B200.
"""
import itertools

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2505_21194_b200 as sc  # noqa: E402


def _sp(p: oracle.Params) -> sc.SeqParams:
    # the two sides keep separate parameter types on purpose (no shared code)
    return sc.SeqParams(p.mode, p.seq_length, p.skip_trigger, p.skip_size, p.min_size, p.max_size,
                        (sc.FLAG_SIGNED if p.signed else 0) | (sc.FLAG_PAIRS if p.pairs else 0))


def _dev(b: np.ndarray):
    return torch.from_numpy(np.ascontiguousarray(b)).cuda()


def _gpu_chunk(b: np.ndarray, p: oracle.Params, offset: int = 0) -> np.ndarray:
    if offset:
        buf = torch.zeros(b.size + offset, dtype=torch.uint8, device="cuda")
        buf[offset:] = _dev(b)
        d = buf[offset:]
    else:
        d = _dev(b)
    return sc.chunk(d, _sp(p)).cpu().numpy().astype(np.uint64)


def _gpu_batch(b: np.ndarray, offs: np.ndarray, p: oracle.Params):
    cuts, idx = sc.chunk_batch(_dev(b), torch.from_numpy(offs.astype(np.int64)).cuda(), _sp(p))
    return cuts.cpu().numpy().astype(np.uint64), idx.cpu().numpy().astype(np.uint64)


def _assert_same(got, want, what=""):
    got = np.asarray(got, dtype=np.uint64)
    want = np.asarray(want, dtype=np.uint64)
    if got.shape != want.shape or not np.array_equal(got, want):
        n = min(got.size, want.size)
        bad = np.nonzero(got[:n] != want[:n])[0]
        first = int(bad[0]) if bad.size else n
        raise AssertionError(f"{what}: len gpu={got.size} oracle={want.size}; first mismatch at {first}: "
                             f"gpu={got[first:first + 4]} oracle={want[first:first + 4]}")


@pytest.fixture(autouse=True)
def _reset_segments():
    sc.set_segment_bytes(0)
    yield
    sc.set_segment_bytes(0)


@pytest.fixture(params=["warp", "lane"])
def walker(request, monkeypatch):
    """Run a single-stream test on both walkers: the warp-cooperative dense one
    and the per-lane sparse one (seqcdc_lane.cuh; it takes M <= 4 runs only,
    other parameter sets stay on the warp walker)."""
    monkeypatch.setenv("SEQCDC_WALKER", request.param)
    return request.param


# ------------------------------------------------------------------ exhaustive tiny inputs
GRID = [(2, 2, 2, 1, 0), (2, 2, 3, 1, 1), (2, 3, 5, 2, 0), (3, 3, 4, 2, 0), (3, 4, 7, 1, 3),
        (3, 5, 8, 3, 1), (4, 4, 8, 2, 1)]


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("L,mn,mx,T,S", GRID)
def test_bruteforce_batch(mode, L, mn, mx, T, S):
    """Every string over {0,1,2} up to length 8, each its own stream of one batch."""
    p = oracle.Params(mode, L, T, S, mn, mx)
    strings = [np.array(t, np.uint8) for n in range(9) for t in itertools.product((0, 1, 2), repeat=n)]
    offs = np.zeros(len(strings) + 1, np.uint64)
    offs[1:] = np.cumsum([s.size for s in strings])
    allb = np.concatenate(strings)
    want_c, want_i = oracle.chunk_batch(allb, offs, p)
    got_c, got_i = _gpu_batch(allb, offs, p)
    _assert_same(got_i, want_i, "cut_index")
    _assert_same(got_c, want_c, "cuts")


# ------------------------------------------------------------------ randomized
def _random_stream(rng, n):
    alpha = int(rng.choice([2, 3, 4, 8, 256]))
    b = rng.integers(0, alpha, n).astype(np.uint8)
    for _ in range(int(rng.integers(0, 8))):
        if n < 3:
            break
        s = int(rng.integers(0, n - 2))
        ln = int(rng.integers(2, min(600, n - s) + 1))
        b[s:s + ln] = (int(rng.integers(0, 256)) + (1 if rng.random() < .5 else -1) * np.arange(ln)) % 256
    return b


def test_randomized_batches():
    rng = np.random.default_rng(2025)
    for trial in range(40):
        L = int(rng.integers(2, 17))
        mn = int(rng.integers(L, L + 400))
        mx = int(rng.integers(mn, mn + 900))
        p = oracle.Params(int(rng.integers(0, 2)), L, int(rng.integers(1, 70)), int(rng.integers(0, 400)), mn, mx)
        streams = [_random_stream(rng, int(rng.integers(0, 30000))) for _ in range(60)]
        offs = np.zeros(len(streams) + 1, np.uint64)
        offs[1:] = np.cumsum([s.size for s in streams])
        allb = np.concatenate(streams)
        want_c, want_i = oracle.chunk_batch(allb, offs, p)
        got_c, got_i = _gpu_batch(allb, offs, p)
        _assert_same(got_i, want_i, f"trial {trial} cut_index {p}")
        _assert_same(got_c, want_c, f"trial {trial} cuts {p}")


# ------------------------------------------------------------------ single streams, all data shapes
KIND_CASES = [
    ("uniform", 1, 8 << 20, oracle.table1(8)),                 # BASELINE config 1
    ("markov", 2, 48 << 20, oracle.table1(4, 1)),              # config 2 shape, scaled
    ("zeroheavy", 3, 32 << 20, oracle.table1(8)),
    ("rampmix", 5, 32 << 20, oracle.table1(8)),
    ("uniform", 7, 24 << 20, oracle.table1(16)),
    ("markov", 9, 16 << 20, oracle.table1(16, 0)),
]


@pytest.mark.parametrize("kind,seed,n,p", KIND_CASES)
def test_single_stream_kinds(kind, seed, n, p, walker):
    b = synth.fill_host(kind, seed, 0, n)
    want = oracle.chunk(b, p)
    _assert_same(_gpu_chunk(b, p), want, kind)


@pytest.mark.parametrize("G", [1 << 16, 3 << 16, 1 << 20, 5 << 20])
@pytest.mark.parametrize("kind,p", [("uniform", oracle.table1(8)), ("markov", oracle.table1(4, 1)),
                                    ("rampmix", oracle.table1(8)), ("zeroheavy", oracle.table1(16)),
                                    ("uniform", oracle.table1(16))])
def test_segment_size_independence(G, kind, p, walker):
    """Cut lists do not depend on the speculative segment length (many seams,
    extensions spanning several segments)."""
    b = synth.fill_host(kind, 11, 0, 12 << 20)
    want = oracle.chunk(b, p)
    sc.set_segment_bytes(G)
    _assert_same(_gpu_chunk(b, p), want, f"{kind} G={G}")


@pytest.mark.parametrize("name", ["zeros", "const7", "inc_ramp", "dec_ramp", "alt2", "sawtooth"])
@pytest.mark.parametrize("G", [0, 1 << 16])
def test_phase_locked_and_degenerate(name, G, walker):
    n = 6 << 20
    i = np.arange(n)
    b = {"zeros": np.zeros(n), "const7": np.full(n, 7), "inc_ramp": i % 256, "dec_ramp": (255 - i) % 256,
         "alt2": i % 2, "sawtooth": (i % 37) * 7}[name].astype(np.uint8)
    sc.set_segment_bytes(G)
    for p in (oracle.table1(8), oracle.table1(4, 1), oracle.Params(0, 3, 1, 0, 64, 64)):
        _assert_same(_gpu_chunk(b, p), oracle.chunk(b, p), f"{name} {p}")


@pytest.mark.parametrize("offset", list(range(1, 16)))
def test_unaligned_input(offset, walker):
    b = synth.fill_host("rampmix", 100 + offset, 0, (1 << 20) + offset * 7)
    p = oracle.table1(8)
    _assert_same(_gpu_chunk(b, p, offset=offset), oracle.chunk(b, p), f"offset {offset}")


def test_edge_sizes(walker):
    p = oracle.Params(0, 5, 50, 256, 4096, 16384)
    L, mn, mx = p.seq_length, p.min_size, p.max_size
    for n in [0, 1, 2, L - 1, L, L + 1, mn - 1, mn, mn + 1, mx - 1, mx, mx + 1, 2 * mx + 3, 3 * TILE_HINT + 5]:
        b = synth.fill_host("uniform", n + 3, 0, n)
        _assert_same(_gpu_chunk(b, p), oracle.chunk(b, p), f"n={n}")


TILE_HINT = 2048


def test_parameter_extremes(walker):
    rng = np.random.default_rng(5)
    b = _random_stream(rng, 300_000)
    for p in [oracle.Params(0, 2, 1, 0, 2, 2), oracle.Params(1, 16, 1, 1000, 16, 16),
              oracle.Params(0, 16, 200, 3, 16, 5000), oracle.Params(1, 2, 10**6, 0, 2, 100000),
              oracle.Params(0, 5, 1, 100000, 5, 70000), oracle.Params(0, 9, 3, 17, 300, 301)]:
        _assert_same(_gpu_chunk(b, p), oracle.chunk(b, p), str(p))


def test_batch_config3_scaled():
    """BASELINE config 3 shape, scaled: 48 streams x 2 MiB +-25% (odd sizes),
    50/30/20 uniform/Markov/zero-heavy, Table I sweep."""
    allb, offs = synth.batch_host(3, 48, 2 << 20)
    for avg in (4, 8, 16):
        p = oracle.table1(avg)
        want_c, want_i = oracle.chunk_batch(allb, offs, p)
        got_c, got_i = _gpu_batch(allb, offs, p)
        _assert_same(got_i, want_i, f"avg {avg} cut_index")
        _assert_same(got_c, want_c, f"avg {avg} cuts")


def test_config2_full_size():
    """BASELINE config 2 at full size (1 GiB Markov, Decreasing, 4 KiB params),
    generated on the device, every cut compared with the oracle."""
    n = 1 << 30
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    synth.fill_device("markov", 2, 0, d)
    p = oracle.table1(4, 1)
    got = sc.chunk(d, _sp(p)).cpu().numpy().astype(np.uint64)
    b = d.cpu().numpy()
    # spot-check generator agreement host vs device on a few blocks
    for pos in (0, 12345678, n - 70000):
        assert np.array_equal(synth.fill_host("markov", 2, pos, 70000), b[pos:pos + 70000])
    _assert_same(got, oracle.chunk(b, p), "config 2")


def test_stream_over_4gib():
    """A single stream longer than 2^32 bytes (positions re-based inside the
    walker; the north-star >= 4 GiB case), config-5 data shape, every cut
    compared with the oracle."""
    n = (4 << 30) + (3 << 20) + 12345
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    synth.fill_device("rampmix", 5, 0, d)
    p = oracle.table1(8)
    got = sc.chunk(d, _sp(p)).cpu().numpy().astype(np.uint64)
    b = d.cpu().numpy()
    del d
    _assert_same(got, oracle.chunk(b, p), "4 GiB+")


def _flat_runs_stream(rng, n):
    """Random pieces separated by runs of one repeated byte (length 1..6000):
    exercises the walker's equal-bytes gallop entering/leaving at every offset."""
    out, tot = [], 0
    while tot < n:
        if rng.random() < 0.5:
            ln = int(rng.integers(1, 6000))
            piece = np.full(ln, int(rng.integers(0, 256)), np.uint8)
        else:
            ln = int(rng.integers(1, 3000))
            piece = rng.integers(0, int(rng.choice([3, 256])), ln).astype(np.uint8)
        out.append(piece)
        tot += ln
    return np.concatenate(out)[:n]


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_flat_runs_gallop(seed):
    rng = np.random.default_rng(seed)
    b = _flat_runs_stream(rng, 3 << 20)
    for p in (oracle.table1(4), oracle.table1(8, 1), oracle.table1(16), oracle.Params(0, 3, 2, 5, 100, 700),
              oracle.Params(1, 6, 9, 0, 64, 5000)):
        _assert_same(_gpu_chunk(b, p), oracle.chunk(b, p), f"flat runs {p}")
    sc.set_segment_bytes(1 << 16)
    p = oracle.table1(4)
    _assert_same(_gpu_chunk(b, p), oracle.chunk(b, p), "flat runs, 64 KiB segments")


@pytest.mark.parametrize("kind,seed", [("uniform", 41), ("markov", 42), ("rampmix", 43)])
def test_signed_flag(kind, seed):
    """SEQCDC_FLAG_SIGNED (int8 byte order, DESIGN.md c6 alternative) against the
    oracle's signed reading, single stream and batch."""
    import dataclasses
    b = synth.fill_host(kind, seed, 0, 6 << 20)
    for p0 in (oracle.table1(8), oracle.table1(4, 1), oracle.Params(0, 3, 4, 9, 40, 400)):
        p = dataclasses.replace(p0, signed=True)
        want = oracle.chunk(b, p)
        _assert_same(_gpu_chunk(b, p), want, f"signed {p}")
        if kind == "uniform":          # (Markov text is 7-bit ASCII: both orders agree there)
            assert not np.array_equal(want, oracle.chunk(b, p0))
    offs = np.array([0, 1000, 500000, 2 << 20, 6 << 20], np.uint64)
    p = dataclasses.replace(oracle.table1(8), signed=True)
    wc, wi = oracle.chunk_batch(b, offs, p)
    gc, gi = _gpu_batch(b, offs, p)
    _assert_same(gi, wi, "signed batch index")
    _assert_same(gc, wc, "signed batch")


@pytest.mark.parametrize("G", [1 << 14, 1 << 16])
def test_batch_overflowing_extensions(G):
    """Batch path: phase-locked streams (no common cut between a chain started
    at a segment start and the true chain) with small segments, so extensions
    exhaust their budget and k_stitch continues them; mixed with normal
    streams and empty ones."""
    rng = np.random.default_rng(G)
    n = 700_000
    i = np.arange(n)
    streams = [((255 - i) % 256).astype(np.uint8),                 # descending ramp (Increasing mode)
               np.full(n // 2 + 7, 9, np.uint8),
               synth.fill_host("uniform", 5, 0, n),
               np.zeros(0, np.uint8),
               ((255 - i[: n // 3]) % 256).astype(np.uint8)]
    offs = np.zeros(len(streams) + 1, np.uint64)
    offs[1:] = np.cumsum([s.size for s in streams])
    allb = np.concatenate(streams)
    sc.set_segment_bytes(G)
    for p in (oracle.Params(0, 5, 50, 256, 1000, 4000), oracle.Params(0, 4, 3, 40, 300, 1111)):
        want_c, want_i = oracle.chunk_batch(allb, offs, p)
        got_c, got_i = _gpu_batch(allb, offs, p)
        _assert_same(got_i, want_i, f"cut_index {p}")
        _assert_same(got_c, want_c, f"cuts {p}")


@pytest.mark.parametrize("kind,seed", [("uniform", 51), ("markov", 52), ("zeroheavy", 53)])
def test_pairs_flag(kind, seed):
    """SEQCDC_FLAG_PAIRS (SeqLength counts comparisons, DESIGN.md c1 alternative)
    against the oracle's comparisons reading: L = 4 (the 4-pair fast path), 5
    and 9 (general run masks), 2 (short runs), single stream and batch."""
    import dataclasses
    b = synth.fill_host(kind, seed, 0, 6 << 20)
    for p0 in (oracle.table1(4, 1), oracle.table1(8), oracle.Params(0, 4, 50, 256, 4096, 16384),
               oracle.Params(1, 9, 30, 100, 2048, 8192), oracle.Params(0, 2, 7, 33, 300, 2000)):
        p = dataclasses.replace(p0, pairs=True)
        want = oracle.chunk(b, p)
        _assert_same(_gpu_chunk(b, p), want, f"pairs {p}")
    offs = np.array([0, 777, 400000, 3 << 20, 6 << 20], np.uint64)
    p = dataclasses.replace(oracle.table1(8), pairs=True)
    wc, wi = oracle.chunk_batch(b, offs, p)
    gc, gi = _gpu_batch(b, offs, p)
    _assert_same(gi, wi, "pairs batch index")
    _assert_same(gc, wc, "pairs batch")


def test_concurrent_calls_on_streams():
    """Calls are reentrant: single-stream and batch calls enqueued on four CUDA
    streams at once (each with its own stream-ordered workspace from the
    library's pool, some with caller workspaces) all equal the oracle."""
    kinds = [("uniform", 71, oracle.table1(8)), ("markov", 72, oracle.table1(4, 1)),
             ("rampmix", 73, oracle.table1(16)), ("zeroheavy", 74, oracle.table1(4))]
    n = 12 << 20
    streams = [torch.cuda.Stream() for _ in kinds]
    host = [synth.fill_host(k, s, 0, n) for k, s, _ in kinds]
    outs = []
    torch.cuda.synchronize()
    for rep in range(3):
        for j, ((k, s, p), st) in enumerate(zip(kinds, streams)):
            with torch.cuda.stream(st):
                d = _dev(host[j])
                sp = _sp(p)
                cuts = torch.empty(sc.max_cuts(n, sp), dtype=torch.int64, device="cuda")
                nc = torch.zeros(1, dtype=torch.int64, device="cuda")
                ws = torch.empty(sc.workspace_size(n, 1, sp), dtype=torch.uint8, device="cuda") if j % 2 else None
                sc.chunk_into(d, sp, cuts, nc, workspace=ws, stream=st)
                outs.append((j, cuts, nc, d, ws))
    torch.cuda.synchronize()
    want = [oracle.chunk(h, p) for h, (_, _, p) in zip(host, kinds)]
    for j, cuts, nc, _, _ in outs:
        _assert_same(cuts[: int(nc.item())].cpu().numpy(), want[j], f"stream {j}")


@pytest.mark.parametrize("G", [1 << 14, 1 << 16])
@pytest.mark.parametrize("kind,p", [("uniform", oracle.table1(8)), ("markov", oracle.table1(4, 1)),
                                    ("uniform", oracle.table1(16)), ("rampmix", oracle.Params(0, 5, 103, 7, 5, 21))])
def test_forced_overflows(G, kind, p, walker, monkeypatch):
    """An extension budget of one segment (SEQCDC_EXT_SEGS=1, a testing knob)
    with short segments: most extensions run out of budget, so the valid path is
    continued by fix_overflows / k_stitch (and, on the lane walker, by the
    hand-off warps running concurrently with the lanes); the lists must still
    equal the oracle's.  Single stream and batch."""
    monkeypatch.setenv("SEQCDC_EXT_SEGS", "1")
    b = synth.fill_host(kind, 91, 0, 10 << 20)
    sc.set_segment_bytes(G)
    _assert_same(_gpu_chunk(b, p), oracle.chunk(b, p), f"{kind} G={G} single")
    offs = np.array([0, 3 << 20, (3 << 20) + 12345, 10 << 20], np.uint64)
    want_c, want_i = oracle.chunk_batch(b, offs, p)
    got_c, got_i = _gpu_batch(b, offs, p)
    _assert_same(got_c, want_c, f"{kind} G={G} batch")


@pytest.mark.parametrize("knobs", [{"SEQCDC_LW_LATE_PCT": "50"}, {"SEQCDC_LW_LATE_EXT_PCT": "50"},
                                   {"SEQCDC_LW_LATE_PCT": "10", "SEQCDC_LW_LATE_EXT_PCT": "10", "SEQCDC_LW_EXT_CAP": "4"}])
@pytest.mark.parametrize("G", [1 << 16, 1 << 18])
@pytest.mark.parametrize("kind,p", [("rampmix", oracle.table1(8)), ("markov", oracle.table1(4, 1)),
                                    ("uniform", oracle.table1(4))])
def test_lane_late_handoffs(knobs, G, kind, p, monkeypatch):
    """The lane walker's optional late hand-offs (off by default, measured
    slower): once a share of the lanes finished their speculative part, a lane
    still in it hands the rest of its segment to a warp (lw_serve's TASK_SPEC,
    claimed by a queue warp or by a warp waiting on that segment), and a lane in
    its extension hands that over at its next cut.  The cut lists must still
    equal the oracle's."""
    monkeypatch.setenv("SEQCDC_WALKER", "lane")
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    b = synth.fill_host(kind, 93, 0, 12 << 20)
    sc.set_segment_bytes(G)
    _assert_same(_gpu_chunk(b, p), oracle.chunk(b, p), f"{kind} G={G} {knobs}")
