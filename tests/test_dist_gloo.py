"""The multi-GPU sharding protocol (paper_2505_21194_b200/dist.py) over real
torch.distributed process groups on the CPU (gloo, world_size 2..4), with the
oracle-based range backend: the concatenated per-rank cut lists must equal the
single-stream oracle cut list exactly, including on phase-locked data where
the seam re-synchronisation needs several exchange rounds."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth

CASES = {
    # name: (bytes builder, params, range lengths as fractions or explicit)
    "uniform8k": (lambda: synth.fill_host("uniform", 21, 0, 3 << 20), oracle.table1(8)),
    "markov4k_dec": (lambda: synth.fill_host("markov", 22, 0, 2 << 20), oracle.table1(4, 1)),
    "rampmix8k": (lambda: synth.fill_host("rampmix", 23, 0, 2 << 20), oracle.table1(8)),
    # phase-locked: constant data -> cuts at k*max; a range start that is not a
    # multiple of max never merges, so overhang changes cascade over ranks
    "zeros": (lambda: np.zeros((1 << 20) + 12345, np.uint8), oracle.table1(8)),
    # strictly decreasing bytes in Increasing mode: forced cuts + skips everywhere
    "dec_ramp": (lambda: ((255 - np.arange((1 << 20) + 777)) % 256).astype(np.uint8), oracle.Params(0, 5, 3, 40, 4096, 16384)),
}


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _bounds(n, P, max_size, uneven):
    if uneven:
        w = np.arange(1, P + 1, dtype=np.float64)
        cuts = np.floor(np.cumsum(w) / w.sum() * n).astype(np.int64)
    else:
        cuts = np.array([(n * (k + 1)) // P for k in range(P)], dtype=np.int64)
    b = [0] + cuts.tolist()
    b[-1] = n
    for k in range(1, P):               # every non-final range holds >= max bytes
        b[k] = max(b[k], b[k - 1] + max_size)
    assert b[P - 1] < n
    return b


def _worker(rank, P, port, case, uneven, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=P)
    try:
        from paper_2505_21194_b200.dist import Shard, chunk_sharded
        from tests.oracle_range import OracleRangeBackend
        build, p = CASES[case]
        b = build()
        n = b.size
        R = _bounds(n, P, p.max_size, uneven)
        lo, hi = R[rank], R[rank + 1]
        end = n if rank == P - 1 else min(n, hi + p.max_size)
        shard = Shard(b[lo:end], hi - lo, lo, n)
        res = chunk_sharded(shard, OracleRangeBackend(p))
        cuts = [int(c) for c in np.asarray(res.cuts)[: res.count]]
        allc = [None] * P
        dist.all_gather_object(allc, (rank, res.first_index, res.total, res.rounds, cuts))
        if rank == 0:
            q.put(allc)
    finally:
        dist.destroy_process_group()


RUNS = [(2, c) for c in CASES] + [(3, "markov4k_dec"), (3, "zeros"), (3, "dec_ramp"), (4, "uniform8k"), (4, "zeros"),
                                   (8, "uniform8k"), (8, "zeros"), (8, "dec_ramp")]


@pytest.mark.parametrize("P,case", RUNS)
def test_sharded_equals_single_stream(P, case):
    if case in ("zeros", "dec_ramp") and P == 3:
        uneven = True
    else:
        uneven = P == 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, P, port, case, uneven, q)) for r in range(P)]
    for pr in procs:
        pr.start()
    allc = q.get(timeout=240)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    build, p = CASES[case]
    want = oracle.chunk(build(), p)
    got = []
    for rank, first, total, rounds, cuts in sorted(allc):
        assert first == len(got), (rank, first, len(got))
        got += cuts
        assert total == want.size
    assert np.array_equal(np.asarray(got, np.uint64), want), case
    if case == "zeros" and P >= 3:
        assert max(r[3] for r in allc) >= 2      # overhang changes cascaded (several rounds)


def _halo_worker(rank, P, port, halo, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=P)
    try:
        from paper_2505_21194_b200.dist import Shard, chunk_sharded
        from tests.oracle_range import OracleRangeBackend
        p = oracle.table1(8)
        b = synth.fill_host("uniform", 31, 0, 1 << 20)
        lo, hi = (0, 1 << 19) if rank == 0 else (1 << 19, 1 << 20)
        end = min(b.size, hi + halo) if rank == 0 else b.size
        err = ""
        if rank == 0:                  # the check runs before any collective
            try:
                chunk_sharded(Shard(b[lo:end], hi - lo, lo), OracleRangeBackend(p))
            except ValueError as e:
                err = str(e)
        q.put((rank, err))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("halo,raises", [(0, True), (16382, True)])
def test_non_final_range_needs_a_right_halo(halo, raises):
    """A non-final range without max_size - 1 bytes past its end would take the
    buffer end for the stream end and force a cut there: refused."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_halo_worker, args=(r, 2, port, halo, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=240) for _ in range(2))
    for pr in procs:
        pr.join(timeout=60)
    assert bool(res[0]) == raises, res


def test_lpt_assign_balances_and_partitions():
    from paper_2505_21194_b200.dist import lpt_assign
    rng = np.random.default_rng(4)
    sizes = rng.integers(1, 1 << 26, 256)
    for P in (1, 2, 3, 8):
        parts = lpt_assign(sizes, P)
        flat = sorted(j for part in parts for j in part)
        assert flat == list(range(sizes.size))                        # every stream exactly once
        loads = [int(sizes[part].sum()) for part in parts]
        assert max(loads) - min(loads) <= int(sizes.max())            # LPT bound: gap <= largest job
    assert lpt_assign([5, 5, 5], 2) == [[0, 2], [1]]


def _p2p_agree_worker(rank, P, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=P)
    try:
        import paper_2505_21194_b200 as sc
        from paper_2505_21194_b200.dist import CudaRangeBackend
        be = CudaRangeBackend(sc.SeqParams.table1(8), device="cuda:0")
        ok = be.enable_p2p()
        res = [None] * P
        dist.all_gather_object(res, (rank, ok, be.p2p, getattr(be, "p2p_error", "")))
        if rank == 0:
            q.put(res)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("P", [2, 3])
def test_p2p_mode_agreement_without_gpu(P):
    """The fused exchange is switched on only if every rank mapped its peer's
    mailbox: here (no GPU) every allocation fails, each rank's error reaches all
    ranks and all of them stay on the collective exchange (no rank is left in
    the fused protocol while another waits in an all_gather)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("needs a box without a GPU (with one, the mailboxes map; see test_gpu_range.py p2p cases)")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_p2p_agree_worker, args=(r, P, port, q)) for r in range(P)]
    for pr in procs:
        pr.start()
    res = q.get(timeout=240)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert len(res) == P
    for rank, ok, p2p, err in res:
        assert ok is False and p2p is False and err, (rank, ok, p2p, err)
