"""Pins for the CPU oracle (oracle/): it is checked against things other than
itself -- the paper's worked example, SPEC's example,
closed forms on data whose cuts follow from the definition by hand, the
mathematics of the method (partition, bounds, witnesses, mode symmetry,
prefix stability, shift equivariance), an independently written query
formulation on exhaustive tiny inputs, and the survey's
Monte-Carlo statistics (SURVEY.md Appendix A [MC-2]).

All tests here are CPU-only (-m "not gpu").
"""
import itertools

import numpy as np
import pytest

import oracle
from oracle import Params, INCREASING, DECREASING


def _golden_params(g):
    return Params(int(g["mode"][0]), int(g["seq_length"][0]), int(g["skip_trigger"][0]),
                  int(g["skip_size"][0]), int(g["min_size"][0]), int(g["max_size"][0]))


def _golden_bytes(g):
    return np.array([int(h, 16) for h in g["bytes"]], dtype=np.uint8)


# ---------------------------------------------------------------- worked examples
def test_fig3_worked_example(golden):
    """L=3, bits 61 of M1 and M2 set -> boundary 3 bytes ahead = 64."""
    g = golden("fig3_block.txt")
    b, p = _golden_bytes(g), _golden_params(g)
    assert b.size == 66 and list(b[:2]) == [0xAF, 0x41]
    assert list(b[61:66]) == [0x12, 0x13, 0x14, 0x11, 0xA4]
    cuts = oracle.chunk(b, p)
    assert int(cuts[0]) == int(g["first_cut"][0]) == 61 + 3
    assert oracle.chunk_py(b, p)[0] == 64
    # Reading c1 (SeqLength counts BYTES): under the "SeqLength comparisons"
    # reading (equivalent to seq_length = L+1 here) there is no boundary in the block.
    p_pairs = Params(p.mode, p.seq_length + 1, p.skip_trigger, p.skip_size, p.min_size + 1,
                     p.max_size)
    assert list(oracle.chunk(b, p_pairs)) == [66]
    # Reading c6 (UNSIGNED bytes): a signed compare would cut at 63 (F0 = -16 < 0x12).
    signed = (b.astype(np.int16) ^ 0x80).astype(np.uint8)   # signed order == unsigned order of b^0x80
    assert int(oracle.chunk(signed, p)[0]) == 63


def test_spec_example(golden):
    g = golden("spec_example.txt")
    b, p = _golden_bytes(g), _golden_params(g)
    want = [int(x) for x in g["cuts"]]
    assert list(oracle.chunk(b, p)) == want == [5, 7]
    assert oracle.chunk_py(b, p) == want
    assert list(oracle.chunk_query(b, p)) == want


def test_spec_all_decreasing_is_max_forced():
    """strictly decreasing everywhere, Increasing mode -> MaxForced at max."""
    n = 10_000
    b = (200 - np.arange(n)) % 256        # one 0->255 step per 256 bytes; no 2 increasing pairs
    for T, S in [(1, 0), (2, 4), (50, 256), (10**9, 0)]:
        p = Params(INCREASING, 3, T, S, 64, 300)
        want = list(range(300, n, 300)) + [n]
        assert list(oracle.chunk(b.astype(np.uint8), p)) == want


def test_spec_descending_ramp_skip_landing():
    """descending ramp, T=2, S=4: the skip lands 4 bytes past the second
    byte of the 2nd decreasing pair, i.e. the scan resumes at pair (3+4)."""
    b = np.array([9, 8, 7, 6, 5, 4, 3, 20, 21, 22, 23, 24], dtype=np.uint8)
    p = Params(INCREASING, 3, 2, 4, 3, 100)
    # pairs (9,8)#1 (8,7)#2 -> d=1, resume at a = d+1+S = 6: bytes 3,20,21 -> cut 9
    assert list(oracle.chunk(b, p))[0] == 9


# ---------------------------------------------------------------- readings c2/c3/c4
def test_skip_landing_discriminates_readings():
    """Data built so that each alternative reading of P:189/P:227 gives a
    different first cut: adopted (reach T, land d+1+S) -> 9; land at d+S -> 8;
    land at d+2+S -> 12; 'exceeds T' -> 5."""
    b = np.array([5, 4, 3, 7, 8, 9, 10, 11, 12, 0, 1, 2], dtype=np.uint8)
    p = Params(INCREASING, 3, 2, 4, 3, 100)
    assert list(oracle.chunk(b, p)) == [9, 12]
    # reading 'exceeds T' == reaching T+1 (c2)
    assert list(oracle.chunk(b, Params(INCREASING, 3, 3, 4, 3, 100)))[0] == 5
    # landing one byte earlier / later == S-1 / S+1 under the adopted rule
    assert list(oracle.chunk(b, Params(INCREASING, 3, 2, 3, 3, 100)))[0] == 8
    assert list(oracle.chunk(b, Params(INCREASING, 3, 2, 5, 3, 100)))[0] == 12


def test_opposing_count_survives_run_breaks():
    """c4: favourable pairs do not reset the opposing counter."""
    b = np.array([5, 4, 6, 5, 7, 6, 7, 8, 9, 10, 0, 0, 0], dtype=np.uint8)
    p = Params(INCREASING, 4, 3, 1, 4, 100)
    # O at pairs 0,2,4 -> third O at d=4 -> resume at 6: 7,8,9,10 -> cut 10
    assert list(oracle.chunk(b, p)) == [10, 13]


def test_equal_bytes_neither():
    """c5: equal bytes neither extend a run nor count as opposing pairs."""
    b = np.array([1, 1, 1, 1, 1, 2, 3, 4, 4], dtype=np.uint8)
    # T=1: any opposing pair would skip 100 bytes (-> cut at n); none exists
    p = Params(INCREASING, 4, 1, 100, 4, 100)
    assert list(oracle.chunk(b, p)) == [8, 9]


def test_skip_past_limit_gives_limit():
    b = np.array([9, 8, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10], dtype=np.uint8)
    p = Params(INCREASING, 3, 1, 50, 3, 8)
    # T=1: pair (9,8) triggers a skip to 0+1+50 > limit 8 -> forced cut at 8 (c8)
    assert list(oracle.chunk(b, p)) == [8, 11, 12]


# ---------------------------------------------------------------- closed forms
def _ramp_cuts(n, c, p, T_is_one=False):
    """Cuts of b[i] = (c+i) mod 256 in Increasing mode, derived by hand: every
    pair is favourable except the wrap pair w (b[w]=255); the run anchored at
    a = base+min-L completes at a+L unless a wrap lies in pairs a..a+L-2, in
    which case the run restarts at w+1 and completes at w+1+L (or, with T=1,
    the wrap triggers a skip and the run starts at w+1+S)."""
    L, cuts, base = p.seq_length, [], 0
    while base < n:
        limit = min(base + p.max_size, n)
        a = base + p.min_size - L
        w = a + ((255 - (c + a)) % 256)           # first wrap pair at or after a
        if w <= a + L - 2:
            start = w + 1 + (p.skip_size if T_is_one else 0)
            cand = start + L
        else:
            cand = a + L
        cut = cand if cand <= limit else limit
        cuts.append(cut)
        base = cut
    return cuts


@pytest.mark.parametrize("c", [0, 3, 200, 255])
@pytest.mark.parametrize("L,mn,mx", [(2, 2, 2), (3, 7, 40), (5, 64, 300), (5, 253, 600), (7, 300, 300)])
def test_increasing_ramp_closed_form(c, L, mn, mx):
    n = 5000
    b = ((c + np.arange(n)) % 256).astype(np.uint8)
    p = Params(INCREASING, L, 2, 17, mn, mx)
    assert list(oracle.chunk(b, p)) == _ramp_cuts(n, c, p)
    p1 = Params(INCREASING, L, 1, 5, mn, mx)
    assert list(oracle.chunk(b, p1)) == _ramp_cuts(n, c, p1, T_is_one=True)
    # Decreasing mode on the complemented ramp is the same closed form
    pd = Params(DECREASING, L, 2, 17, mn, mx)
    assert list(oracle.chunk(255 - b, pd)) == _ramp_cuts(n, c, p)


@pytest.mark.parametrize("value", [0, 7, 255])
@pytest.mark.parametrize("mode", [INCREASING, DECREASING])
def test_constant_data_is_max_forced(value, mode):
    n = 100_003
    b = np.full(n, value, dtype=np.uint8)
    for p in [oracle.table1(4, mode), oracle.table1(8, mode), oracle.table1(16, mode),
              Params(mode, 2, 1, 0, 2, 2)]:
        want = list(range(p.max_size, n, p.max_size)) + [n]
        assert list(oracle.chunk(b, p)) == want


def test_empty_and_tiny():
    p = oracle.table1(8)
    assert oracle.chunk(np.zeros(0, np.uint8), p).size == 0
    assert list(oracle.chunk(np.array([1], np.uint8), p)) == [1]
    assert list(oracle.chunk(np.arange(10, dtype=np.uint8), Params(INCREASING, 2, 1, 0, 2, 2))) == \
        [2, 4, 6, 8, 10]


# ---------------------------------------------------------------- brute force
GRID = [
    # L, min, max, T, S
    (2, 2, 2, 1, 0), (2, 2, 3, 1, 1), (2, 3, 5, 2, 0), (2, 2, 4, 3, 3),
    (3, 3, 3, 1, 1), (3, 3, 4, 2, 0), (3, 4, 7, 1, 3), (3, 5, 8, 3, 1),
    (3, 3, 6, 2, 2), (4, 4, 8, 2, 1),
]


def _all_strings(maxlen, alphabet=(0, 1, 2)):
    for n in range(maxlen + 1):
        for t in itertools.product(alphabet, repeat=n):
            yield np.array(t, dtype=np.uint8)


@pytest.mark.parametrize("mode", [INCREASING, DECREASING])
@pytest.mark.parametrize("L,mn,mx,T,S", GRID)
def test_bruteforce_literal_vs_query(mode, L, mn, mx, T, S):
    """Every string over {0,1,2} up to length 8: the literal C loop, its Python
    twin and the independent query formulation agree."""
    p = Params(mode, L, T, S, mn, mx)
    strings = list(_all_strings(8))
    offs = np.zeros(len(strings) + 1, dtype=np.uint64)
    offs[1:] = np.cumsum([s.size for s in strings])
    allb = np.concatenate(strings) if strings else np.zeros(0, np.uint8)
    cuts, idx = oracle.chunk_batch(allb, offs, p)
    for j, s in enumerate(strings):
        got = [int(c) - int(offs[j]) for c in cuts[int(idx[j]):int(idx[j + 1])]]
        assert got == oracle.chunk_py(s, p), (s, p)
        if s.size >= 3 and j % 3 == 0:        # the numpy formulation is slower; 1/3 sample
            assert got == [int(c) for c in oracle.chunk_query(s, p)], (s, p)


def _random_case(rng):
    alpha = int(rng.choice([2, 3, 4, 8, 256]))
    n = int(rng.integers(0, 3000))
    b = rng.integers(0, alpha, n).astype(np.uint8)
    # splice ramps so runs and skip triggers straddle everything
    for _ in range(int(rng.integers(0, 6))):
        if n < 3:
            break
        s = int(rng.integers(0, n - 2))
        ln = int(rng.integers(2, min(600, n - s) + 1))
        st = int(rng.integers(0, 256))
        d = 1 if rng.random() < 0.5 else -1
        b[s:s + ln] = (st + d * np.arange(ln)) % 256
    L = int(rng.integers(2, 9))
    mn = int(rng.integers(L, L + 300))
    mx = int(rng.integers(mn, mn + 600))
    T = int(rng.integers(1, 60))
    S = int(rng.integers(0, 300))
    return b, Params(int(rng.integers(0, 2)), L, T, S, mn, mx)


def test_randomized_literal_vs_query():
    rng = np.random.default_rng(12345)
    for _ in range(1500):
        b, p = _random_case(rng)
        c = list(oracle.chunk(b, p))
        assert c == [int(x) for x in oracle.chunk_query(b, p)], p
        if b.size < 400:
            assert c == oracle.chunk_py(b, p)


# ---------------------------------------------------------------- invariants
def _check_invariants(b, p, cuts):
    n = b.size
    cuts = [int(c) for c in cuts]
    if n == 0:
        assert cuts == []
        return
    assert cuts[-1] == n
    assert all(x < y for x, y in zip(cuts, cuts[1:]))
    base = 0
    for k, c in enumerate(cuts):
        size = c - base
        assert size <= p.max_size
        if c != n:
            assert size >= p.min_size
        if c != base + p.max_size and c != n:
            # witness: bytes c-L..c-1 strictly monotone in the mode's direction, inside the chunk
            w = b[c - p.seq_length:c].astype(np.int16)
            dif = np.diff(w)
            assert (dif > 0).all() if p.mode == INCREASING else (dif < 0).all()
            assert c - p.seq_length >= base
        base = c


def test_invariants_random():
    rng = np.random.default_rng(7)
    for _ in range(300):
        b, p = _random_case(rng)
        _check_invariants(b, p, oracle.chunk(b, p))


def test_mode_symmetry():
    rng = np.random.default_rng(8)
    for _ in range(200):
        b, p = _random_case(rng)
        pi = Params(INCREASING, p.seq_length, p.skip_trigger, p.skip_size, p.min_size, p.max_size)
        pd = Params(DECREASING, p.seq_length, p.skip_trigger, p.skip_size, p.min_size, p.max_size)
        assert list(oracle.chunk(b, pi)) == list(oracle.chunk(255 - b, pd))


def test_prefix_stability_and_shift_equivariance():
    rng = np.random.default_rng(9)
    p = oracle.table1(8)
    x = rng.integers(0, 256, 1 << 20).astype(np.uint8)
    cx = oracle.chunk(x, p)
    for _ in range(20):
        q = int(rng.integers(0, x.size))
        y = x.copy()
        y[q:] = rng.integers(0, 256, x.size - q)
        cy = oracle.chunk(y, p)
        assert list(cx[cx <= q]) == list(cy[cy <= q])
    for k in rng.integers(0, cx.size - 1, 10):
        c = int(cx[k])
        assert list(oracle.chunk(x[c:], p) + c) == list(cx[k + 1:])


def test_skip_size_zero_is_no_skipping():
    rng = np.random.default_rng(10)
    for _ in range(200):
        b, p = _random_case(rng)
        p0 = Params(p.mode, p.seq_length, p.skip_trigger, 0, p.min_size, p.max_size)
        pinf = Params(p.mode, p.seq_length, 10**9, 123, p.min_size, p.max_size)
        assert list(oracle.chunk(b, p0)) == list(oracle.chunk(b, pinf))


def test_next_cut_is_chunk_step():
    rng = np.random.default_rng(11)
    b = rng.integers(0, 256, 200_000).astype(np.uint8)
    p = oracle.table1(4, DECREASING)
    cuts = oracle.chunk(b, p)
    prev = 0
    for c in cuts[:50]:
        assert oracle.next_cut(b, prev, p) == int(c)
        prev = int(c)


# ---------------------------------------------------------------- statistics (sanity)
@pytest.mark.parametrize("avg,mean,examined", [(4, 2420, 0.062), (8, 4506, 0.033), (16, 8870, 0.017)])
def test_uniform_statistics_match_survey(avg, mean, examined):
    """SURVEY.md Appendix A [MC-2]: uniform data, Table I params, min=avg/2: mean
    chunk 2.42K / 4.51K / 8.87K, bytes examined 6.2% / 3.3% / 1.7%."""
    rng = np.random.default_rng(2024)
    b = rng.integers(0, 256, 32 << 20, dtype=np.uint8)
    cuts, ex = oracle.chunk(b, oracle.table1(avg), return_examined=True)
    assert abs(b.size / cuts.size / mean - 1) < 0.02
    assert abs(ex / b.size - examined) < 0.006


def test_fingerprint_and_dedup_definitions():
    """The dedup oracle against closed forms: FIPS 180-4 test vectors for the
    SHA-256 step, and a stream built from repeated blocks whose stored bytes are
    known exactly (Eq. 1)."""
    import hashlib
    abc = np.frombuffer(b"abc" + b"x" * 61, dtype=np.uint8)
    fp = oracle.fingerprints(abc, [3, 64])
    assert fp[0].tobytes().hex() == "ba7816bf8f01cfea414140de5dae2223b00361a396177a9cb410ff61f20015ad"
    assert fp[1].tobytes() == hashlib.sha256(b"x" * 61).digest()
    e = oracle.fingerprints(np.zeros(0, np.uint8), [])
    assert e.shape == (0, 32)
    rng = np.random.default_rng(1)
    blocks = [rng.integers(0, 256, 1000 + 7 * i).astype(np.uint8) for i in range(5)]
    order = [0, 1, 0, 2, 1, 3, 4, 4, 0]
    data = np.concatenate([blocks[i] for i in order])
    cuts = np.cumsum([blocks[i].size for i in order])
    first, uniq = oracle.dedup(data, cuts)
    assert first.tolist() == [True, True, False, True, False, True, True, False, False]
    assert uniq == sum(b.size for b in blocks)


def test_signed_reading_is_unsigned_on_flipped_bytes():
    """Flag for reading c6's alternative (signed int8 compares): a signed compare
    of x and y orders exactly like an unsigned compare of x^0x80 and y^0x80, so
    the signed oracle on b must equal the unsigned oracle on b^0x80 (closed form),
    and the three formulations agree under the flag."""
    rng = np.random.default_rng(11)
    for trial in range(200):
        n = int(rng.integers(0, 3000))
        b = rng.integers(0, 256, n).astype(np.uint8)
        L = int(rng.integers(2, 7))
        mn = int(rng.integers(L, L + 60))
        p = oracle.Params(int(rng.integers(0, 2)), L, int(rng.integers(1, 40)), int(rng.integers(0, 90)), mn,
                          int(rng.integers(mn, mn + 300)), True)
        pu = oracle.Params(p.mode, p.seq_length, p.skip_trigger, p.skip_size, p.min_size, p.max_size, False)
        want = oracle.chunk(b ^ np.uint8(0x80), pu)
        assert np.array_equal(oracle.chunk(b, p), want)
        if n <= 600:
            assert oracle.chunk_py(b, p) == want.tolist()
            assert np.array_equal(oracle.chunk_query(b, p), want)


def test_fig3_block_signed_reading(golden):
    """Under the signed reading the Fig. 3-consistent block cuts at
    63 instead of 64: AF/F0 are negative as int8, so the filler's F0 -> 12 step is
    increasing (SURVEY [MC-7]; filler-dependent, which is why c6 stays unsigned)."""
    g = golden("fig3_block.txt")
    b = np.array([int(x, 16) for x in g["bytes"]], np.uint8)
    p = oracle.Params(int(g["mode"][0]), int(g["seq_length"][0]), int(g["skip_trigger"][0]),
                      int(g["skip_size"][0]), int(g["min_size"][0]), int(g["max_size"][0]), True)
    assert int(oracle.chunk(b, p)[0]) == 63


def test_pairs_reading_closed_form_on_a_ramp():
    """Flag for reading c1's alternative (SeqLength counts favourable comparisons,
    P:153): on a strictly increasing stream every pair is favourable, so under
    the bytes reading each chunk is exactly min bytes (anchor base+min-L, run of
    L bytes ends at base+min) and under the comparisons reading min+1 (L
    favourable pairs = L+1 bytes from the same anchor)."""
    b = np.arange(256, dtype=np.uint8)
    for L in (2, 4, 5, 7):
        for mn in (L, 20, 33):
            pb = oracle.Params(0, L, 1000, 0, mn, 64)
            pp = oracle.Params(0, L, 1000, 0, mn, 64, pairs=True)
            wb = list(range(mn, 256, mn)) + [256]
            wp = list(range(mn + 1, 256, mn + 1)) + [256]
            assert oracle.chunk(b, pb).tolist() == wb
            assert oracle.chunk(b, pp).tolist() == wp
            assert oracle.chunk_py(b, pp) == wp
            assert oracle.chunk_query(b, pp).tolist() == wp


def test_pairs_reading_is_bytes_reading_shifted():
    """The comparisons reading with (L, min) examines the same anchor (base+min-L)
    and needs L+1 monotone bytes, i.e. the bytes reading with (L+1, min+1): the
    flag must match that parameter shift exactly, in all three formulations, in
    both modes and with skipping (a dropped +1 on either the run or the anchor
    fails here)."""
    rng = np.random.default_rng(12)
    for trial in range(200):
        n = int(rng.integers(0, 3000))
        alpha = int(rng.choice([2, 3, 8, 256]))
        b = rng.integers(0, alpha, n).astype(np.uint8)
        L = int(rng.integers(2, 7))
        mn = int(rng.integers(L, L + 60))
        mx = int(rng.integers(mn + 1, mn + 300))
        mode, T, S = int(rng.integers(0, 2)), int(rng.integers(1, 40)), int(rng.integers(0, 90))
        pp = oracle.Params(mode, L, T, S, mn, mx, pairs=True)
        pb = oracle.Params(mode, L + 1, T, S, mn + 1, mx)
        want = oracle.chunk(b, pb)
        assert np.array_equal(oracle.chunk(b, pp), want)
        if n <= 600:
            assert oracle.chunk_py(b, pp) == want.tolist()
            assert np.array_equal(oracle.chunk_query(b, pp), want)


# ---------------------------------------------------------------- parameter validation
@pytest.mark.parametrize("bad", [
    dict(mode=2), dict(seq_length=1), dict(seq_length=0), dict(skip_trigger=0),
    dict(seq_length=5, min_size=4), dict(min_size=100, max_size=99),
])
def test_check_params_rejects(bad):
    """The oracle refuses what the method cannot mean: a mode other than
    Increasing/Decreasing, a run shorter than 2 bytes, a skip
    trigger of 0, min < SeqLength (the sub-minimum region min-L would be
    negative) and max < min.  Both the C check and Params.check."""
    base = dict(mode=0, seq_length=5, skip_trigger=50, skip_size=256, min_size=4096, max_size=16384)
    base.update(bad)
    p = oracle.Params(**base)
    assert oracle.check_params_c(p) == 1
    with pytest.raises(ValueError):
        p.check()
    with pytest.raises(ValueError):
        oracle.chunk(np.zeros(10, np.uint8), p)


def test_check_params_accepts_boundaries():
    """Smallest accepted values: L = 2, min = L, max = min, T = 1, S = 0."""
    p = oracle.Params(1, 2, 1, 0, 2, 2)
    assert oracle.check_params_c(p) == 0
    p.check()
    # every chunk is exactly min = max = 2 bytes (P:266 forced cut), last one shorter
    assert oracle.chunk(np.arange(7, dtype=np.uint8), p).tolist() == [2, 4, 6, 7]


# ---------------------------------------------------------------- measurement: bytes the method reads
def test_chunk_window_is_prefix_of_chunk():
    """oracle_chunk_window stops after the first chunk starting beyond last_start
    and otherwise equals oracle_chunk (the windowed whole-list check relies on it)."""
    rng = np.random.default_rng(77)
    b = rng.integers(0, 256, 300_000).astype(np.uint8)
    p = oracle.table1(4)
    full = oracle.chunk(b, p)
    for last_start in (0, 1, 5000, int(full[10]), int(full[10]) + 1, b.size):
        got, _, _ = oracle.chunk_window(b, last_start, p)
        starts = np.concatenate([[0], full[:-1]])
        want = full[: int(np.searchsorted(starts, last_start, side="right"))]
        assert np.array_equal(got, want), last_start


def test_touched_units_match_query_form():
    """Distinct units (1, 32, 128, 512 B) holding a compared byte: the literal
    loop's running count equals the query form's interval union (anchors P:179 /
    d+1+S P:189, deciding pair P:225-227) on random small cases."""
    rng = np.random.default_rng(5)
    for it in range(250):
        n = int(rng.integers(0, 3000))
        b = rng.integers(0, int(rng.choice([2, 3, 4, 256])), n).astype(np.uint8)
        L = int(rng.integers(2, 7))
        mn = int(rng.integers(L, 200))
        p = oracle.Params(int(rng.integers(0, 2)), L, int(rng.integers(1, 20)), int(rng.integers(0, 50)), mn,
                          int(rng.integers(mn, 600)), pairs=bool(rng.integers(0, 2)))
        _, pairs, t = oracle.chunk_window(b, n, p, unit_shifts=(0, 5, 7, 9))
        assert {k: v[0] for k, v in t.items()} == oracle.touched_units_query(b, p, (0, 5, 7, 9)), it
        _, ex = oracle.chunk(b, p, return_examined=True)
        assert pairs == ex


@pytest.mark.parametrize("n", [1, 100, 2044, 2045, 5000, 70_001])
def test_touched_bytes_closed_form_constant(n):
    """Constant data: no pair is favourable or opposing, so every
    chunk compares pairs base+min-L .. limit-2 and is cut at limit: the
    bytes read are [base+min-L, limit) per chunk, limit - base - min + L of them
    (none when fewer than 2 bytes follow the anchor)."""
    p = oracle.table1(4)
    b = np.full(n, 9, np.uint8)
    cuts, _, t = oracle.chunk_window(b, n, p, unit_shifts=(0,))
    want, base = 0, 0
    for c in cuts.tolist():
        span = c - base - p.min_size + p.seq_length     # bytes from the anchor to the limit
        want += span if span >= 2 else 0                 # no pair fits in fewer than 2 bytes
        base = c
    assert t[0][0] == want
