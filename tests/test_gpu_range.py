"""GPU parity of the multi-GPU building blocks (seqcdc_range_chunk /
seqcdc_range_resync) and of the sharded protocol driving them.  One GPU:
ranks are emulated as separate processes on cuda:0 exchanging over gloo --
their kernels never wait on one another, so this is safe on one device."""
import os
import socket

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2505_21194_b200 as sc  # noqa: E402


def _sp(p):
    return sc.SeqParams(p.mode, p.seq_length, p.skip_trigger, p.skip_size, p.min_size, p.max_size,
                        (sc.FLAG_SIGNED if p.signed else 0) | (sc.FLAG_PAIRS if p.pairs else 0))


def _oracle_chain(buf, start, range_len, gofs, p):
    cuts, base = [], start
    while base < range_len:
        c = oracle.next_cut(buf, base, p)
        cuts.append(gofs + c)
        base = c
    return np.asarray(cuts, np.uint64)


CASES = [("uniform", 31, oracle.table1(8)), ("markov", 32, oracle.table1(4, 1)), ("rampmix", 33, oracle.table1(8)),
         ("zeroheavy", 34, oracle.table1(16)),
         # the reading flags go through the range calls too
         ("uniform", 35, oracle.Params(0, 4, 50, 256, 4096, 16384, signed=True, pairs=True))]


@pytest.fixture(params=["warp", "lane"])
def walker(request, monkeypatch):
    """Both walkers behind the range calls (the lane walker hands a range call's
    tail to a warp: seqcdc_lane.cuh lw_serve)."""
    monkeypatch.setenv("SEQCDC_WALKER", request.param)
    return request.param


@pytest.mark.parametrize("kind,seed,p", CASES)
@pytest.mark.parametrize("G", [0, 1 << 16])
def test_range_chunk_and_resync(kind, seed, p, G, walker):
    sc.set_segment_bytes(G)
    try:
        n = 6 << 20
        b = synth.fill_host(kind, seed, 0, n)
        sp = _sp(p)
        for lo, hi in [(0, 2 << 20), (1234567, 3 << 20), (5 << 20, n), (777, 777 + p.max_size)]:
            end = n if hi == n else min(n, hi + p.max_size)
            buf_h = b[lo:end]
            buf = torch.from_numpy(buf_h).cuda()
            cap = sc.range_max_cuts(buf.numel(), hi - lo, sp)
            spec = torch.empty(cap, dtype=torch.int64, device="cuda")
            spec_n = torch.zeros(1, dtype=torch.int64, device="cuda")
            sc.range_chunk_into(buf, hi - lo, 0, lo, sp, spec, spec_n)
            got = spec[: int(spec_n.item())].cpu().numpy().astype(np.uint64)
            assert np.array_equal(got, _oracle_chain(buf_h, 0, hi - lo, lo, p)), (kind, lo, hi)
            # the true chain from the true entry: the oracle's first cut >= lo
            full = oracle.chunk(b, p)
            starts = np.concatenate([[0], full]).astype(np.uint64)
            entry = int(starts[starts >= lo][0])      # first chunk start >= lo
            out = torch.empty(cap, dtype=torch.int64, device="cuda")
            out_n = torch.zeros(1, dtype=torch.int64, device="cuda")
            status = torch.zeros(4, dtype=torch.int64, device="cuda")
            sc.range_resync_into(buf, hi - lo, entry - lo, lo, sp, spec, spec_n, out, out_n, status)
            got = out[: int(out_n.item())].cpu().numpy().astype(np.uint64)
            want = full[(full > entry) & (full <= (full[full >= hi][0] if hi < n else n))]
            assert np.array_equal(got, want), (kind, lo, hi, got[:4], want[:4])
            st = status.cpu().tolist()
            assert st[3] == int(want[-1])
            # resync from a non-cut entry equals the chain from there
            sc.range_resync_into(buf, hi - lo, 1, lo, sp, spec, spec_n, out, out_n, status)
            got = out[: int(out_n.item())].cpu().numpy().astype(np.uint64)
            assert np.array_equal(got, _oracle_chain(buf_h, 1, hi - lo, lo, p))
    finally:
        sc.set_segment_bytes(0)


def test_range_entry_at_end_and_errors():
    p = _sp(oracle.table1(8))
    buf = torch.zeros(100, dtype=torch.uint8, device="cuda")
    cuts = torch.empty(8, dtype=torch.int64, device="cuda")
    nc = torch.full((1,), 7, dtype=torch.int64, device="cuda")
    sc.range_chunk_into(buf, 100, 100, 5, p, cuts, nc)
    assert int(nc.item()) == 0
    with pytest.raises(sc.SeqCDCError):
        sc.range_chunk_into(buf, 100, 101, 5, p, cuts, nc)
    with pytest.raises(sc.SeqCDCError):
        sc.range_chunk_into(buf, 50, 51, 0, p, cuts, nc)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, P, port, kind, seed, n, pidx, q, comm="cpu"):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    if ":" in comm:                        # "<comm>:<walker>" forces the walker behind the range calls
        comm, wk = comm.split(":")
        os.environ["SEQCDC_WALKER"] = wk
    dist.init_process_group("gloo", rank=rank, world_size=P)
    try:
        from paper_2505_21194_b200.dist import CudaRangeBackend, Shard, chunk_sharded
        p = _sp(SHARD_PARAMS[pidx])
        lo, hi = n * rank // P, n * (rank + 1) // P
        end = n if rank == P - 1 else min(n, hi + (CudaRangeBackend.TAIL + 1) * p.max_size)
        buf = torch.empty(end - lo, dtype=torch.uint8, device="cuda")
        if kind == "zeros":
            buf.zero_()
        else:
            synth.fill_device(kind, seed, lo, buf)
        be = CudaRangeBackend(p)
        if comm == "p2p":                  # fused exchange: peer-memory mailboxes (CUDA IPC)
            be.enable_p2p()
            comm = "cuda"
        cd = torch.device(comm)
        res = chunk_sharded(Shard(buf, hi - lo, lo, n), be, comm_device=cd)
        res = chunk_sharded(Shard(buf, hi - lo, lo, n), be, comm_device=cd)   # buffers (and mailboxes) reused
        path = be.last_path
        cuts = res.cuts[: res.count].cpu().numpy().tolist()
        allc = [None] * P
        dist.all_gather_object(allc, (rank, res.first_index, res.total, res.rounds, cuts, path))
        dist.barrier()
        be.close()
        if rank == 0:
            q.put(allc)
    finally:
        dist.destroy_process_group()


SHARD_PARAMS = [oracle.table1(8), oracle.table1(4, 1), oracle.table1(16)]


@pytest.mark.parametrize("P,kind,seed,n,pidx,comm", [(2, "rampmix", 41, 24 << 20, 0, "cpu"),
                                                      (3, "markov", 42, 20 << 20, 1, "cpu"),
                                                      (4, "uniform", 43, 30 << 20, 2, "cpu"),
                                                      (3, "zeros", 0, 5 << 20, 0, "cpu"),
                                                      (3, "markov", 44, 20 << 20, 1, "cuda"),
                                                      (4, "zeros", 0, 5 << 20, 0, "cuda"),
                                                      (2, "markov", 45, 16 << 20, 1, "p2p"),
                                                      (3, "rampmix", 46, 24 << 20, 0, "p2p"),
                                                      (3, "zeros", 0, 5 << 20, 0, "p2p"),
                                                      (8, "rampmix", 47, 24 << 20, 0, "cpu"),
                                                      (8, "markov", 48, 24 << 20, 1, "cuda"),
                                                      (8, "zeros", 0, 8 << 20, 0, "cuda"),
                                                      (8, "uniform", 49, 32 << 20, 0, "p2p"),
                                                      (3, "rampmix", 50, 24 << 20, 0, "p2p:lane"),
                                                      (2, "markov", 51, 16 << 20, 1, "cuda:lane")])
def test_sharded_protocol_on_one_gpu(P, kind, seed, n, pidx, comm):
    """comm="cuda": the device protocol (no host sync inside the round; the
    exchanges run on device tensors), falling back to the host loop on the
    phase-locked stream.  comm="p2p": the fused exchange -- each range's last
    kernel stores its block into the next rank's mailbox (CUDA IPC) and the
    merge kernel waits for the flag on the device; here the ranks share one
    GPU, across GPUs the stores go over NVLink."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, P, port, kind, seed, n, pidx, q, comm)) for r in range(P)]
    for pr in procs:
        pr.start()
    allc = q.get(timeout=600)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    b = np.zeros(n, np.uint8) if kind == "zeros" else synth.fill_host(kind, seed, 0, n)
    want = oracle.chunk(b, SHARD_PARAMS[pidx])
    got = []
    for rank, first, total, rounds, cuts, path in sorted(allc):
        assert first == len(got)
        got += cuts
        assert total == want.size
        if comm.startswith("p2p") and kind != "zeros":   # the fused round settled it (no fallback)
            assert path == "p2p", (rank, path)
    assert np.array_equal(np.asarray(got, np.uint64), want)


@pytest.mark.parametrize("kind,seed,p", CASES)
def test_range_tail_and_local_merge(kind, seed, p, walker):
    """seqcdc_range_chunk_tail's tail = the oracle chain continued past the
    overhang (fully determined chunks only); seqcdc_range_merge_tail on the next
    range = the true chain of that range, whether the tail reaches the merge or
    the re-walk fallback runs (tiny tail_max)."""
    n = 8 << 20
    b = synth.fill_host(kind, seed, 0, n)
    sp = _sp(p)
    R = [0, 3 << 20, n]
    E = 96
    full = oracle.chunk(b, p)
    for tail_max in (E, 2):
        # range 0 with its halo
        end0 = min(n, R[1] + (E + 1) * p.max_size)
        buf0 = torch.from_numpy(b[:end0]).cuda()
        cap0 = sc.range_max_cuts(buf0.numel(), R[1], sp)
        c0 = torch.empty(cap0, dtype=torch.int64, device="cuda")
        n0 = torch.zeros(1, dtype=torch.int64, device="cuda")
        blk = torch.zeros(3 + E, dtype=torch.int64, device="cuda")
        sc.range_chunk_tail_into(buf0, R[1], 0, sp, c0, n0, tail_max, blk)
        k0 = int(n0.item())
        ov = int(c0[k0 - 1].item())
        assert blk[:2].cpu().tolist() == [ov, k0]          # the summary written by the library
        tn = int(blk[2].item())
        tail = blk[3:3 + tn].cpu().numpy().astype(np.uint64)
        # oracle: the true chain from the overhang, chunks wholly inside the buffer
        want_tail = [ov]
        base = ov
        while len(want_tail) < tail_max and base + p.max_size <= end0:
            base = oracle.next_cut(b[:end0], base, p)
            want_tail.append(base)
        assert tail.tolist() == want_tail, (kind, tail_max)
        # range 1: speculative pass + local merge with range 0's tail
        buf1 = torch.from_numpy(b[R[1]:]).cuda()
        cap1 = sc.range_max_cuts(buf1.numel(), R[2] - R[1], sp)
        spec = torch.empty(cap1, dtype=torch.int64, device="cuda")
        spec_n = torch.zeros(1, dtype=torch.int64, device="cuda")
        sc.range_chunk_into(buf1, R[2] - R[1], 0, R[1], sp, spec, spec_n)
        out = torch.empty(cap1, dtype=torch.int64, device="cuda")
        out_n = torch.zeros(1, dtype=torch.int64, device="cuda")
        status = torch.zeros(4, dtype=torch.int64, device="cuda")
        own = torch.tensor([12345], dtype=torch.int64, device="cuda")
        sum3 = torch.zeros(3, dtype=torch.int64, device="cuda")
        sc.range_merge_tail_into(buf1, R[2] - R[1], R[1], sp, blk, E if tail_max == E else tail_max, spec, spec_n,
                                 out, out_n, status, spec_ov=own, sum3=sum3)
        got = out[: int(out_n.item())].cpu().numpy().astype(np.uint64)
        want = full[full > ov]
        assert np.array_equal(got, want), (kind, tail_max, status.cpu().tolist())
        assert sum3.cpu().tolist() == [int(want[-1]), int(want.size), 12345]


def _batch_worker(rank, P, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=P)
    try:
        from paper_2505_21194_b200.dist import chunk_batch_sharded, lpt_assign
        off, kinds, seeds = synth.batch_layout(3, 24, 1 << 20)
        sizes = np.diff(off.astype(np.int64))
        mine = lpt_assign(sizes, P)[rank]
        streams = {}
        for j in mine:
            t = torch.empty(int(sizes[j]), dtype=torch.uint8, device="cuda")
            synth.fill_device(int(kinds[j]), int(seeds[j]), 0, t)
            streams[j] = t
        out, total = chunk_batch_sharded(streams, _sp(oracle.table1(8)))
        res = {j: c.cpu().numpy().tolist() for j, c in out.items()}
        allr = [None] * P
        dist.all_gather_object(allr, (res, total))
        if rank == 0:
            q.put(allr)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("P", [2, 3])
def test_batch_sharded_lpt(P):
    """Batches of independent streams over P ranks (LPT by size, no data-path
    collective): per-stream cut lists = the oracle's, totals all-reduced."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_batch_worker, args=(r, P, port, q)) for r in range(P)]
    for pr in procs:
        pr.start()
    allr = q.get(timeout=600)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    off, kinds, seeds = synth.batch_layout(3, 24, 1 << 20)
    p = oracle.table1(8)
    got = {}
    for res, total in allr:
        got.update(res)
    want_total = 0
    for j in range(24):
        b = synth.fill_host(int(kinds[j]), int(seeds[j]), 0, int(off[j + 1] - off[j]))
        w = oracle.chunk(b, p)
        want_total += w.size
        assert np.array_equal(np.asarray(got[j], np.uint64), w), j
    assert all(t == want_total for _, t in allr)


def test_fused_push_and_wait_single_process():
    """The fused-exchange pieces in one process: seqcdc_range_chunk_tail_push
    stores the block into the given mailbox address and releases the flag;
    seqcdc_range_merge_tail_wait on that mailbox gives the next range's true
    chain (= the oracle), exactly as seqcdc_range_merge_tail on the block; with a
    flag value that never arrives it times out into the collective-fallback
    signal (overhang UINT64_MAX) instead of hanging."""
    p = oracle.table1(8)
    sp = _sp(p)
    n = 8 << 20
    b = synth.fill_host("markov", 61, 0, n)
    full = oracle.chunk(b, p)
    E, R1 = 96, 3 << 20
    end0 = R1 + (E + 1) * p.max_size
    buf0 = torch.from_numpy(b[:end0]).cuda()
    cap0 = sc.range_max_cuts(buf0.numel(), R1, sp)
    c0 = torch.empty(cap0, dtype=torch.int64, device="cuda")
    n0 = torch.zeros(1, dtype=torch.int64, device="cuda")
    blk = torch.zeros(3 + E, dtype=torch.int64, device="cuda")
    mb, handle = sc.xchg_alloc(4096)
    try:
        assert len(handle) == sc.IPC_HANDLE_BYTES
        flag = mb + 2048
        sc.range_chunk_tail_push_into(buf0, R1, 0, sp, c0, n0, E, blk, mb, flag, 7)
        k0 = int(n0.item())
        ov = int(c0[k0 - 1].item())
        assert blk[:2].cpu().tolist() == [ov, k0]
        # the next range: its speculative chain, then the merge from the mailbox
        buf1 = torch.from_numpy(b[R1:]).cuda()
        cap1 = sc.range_max_cuts(buf1.numel(), n - R1, sp)
        spec = torch.empty(cap1, dtype=torch.int64, device="cuda")
        spec_n = torch.zeros(1, dtype=torch.int64, device="cuda")
        own = torch.zeros(3 + E, dtype=torch.int64, device="cuda")
        sc.range_chunk_tail_into(buf1, n - R1, R1, sp, spec, spec_n, 0, own)
        out = torch.empty(cap1, dtype=torch.int64, device="cuda")
        out_n = torch.zeros(1, dtype=torch.int64, device="cuda")
        status = torch.zeros(4, dtype=torch.int64, device="cuda")
        sum3 = torch.zeros(3, dtype=torch.int64, device="cuda")
        sc.range_merge_tail_wait_into(buf1, n - R1, R1, sp, mb, flag, 7, E, spec, spec_n, out, out_n, status,
                                      spec_ov=own, sum3=sum3)
        want = full[full > ov]
        got = out[: int(out_n.item())].cpu().numpy().astype(np.uint64)
        assert np.array_equal(got, want)
        assert sum3.cpu().tolist()[:2] == [int(want[-1]), int(want.size)]
        # a flag value that never arrives: bounded wait, then the fallback signal
        sc.range_merge_tail_wait_into(buf1, n - R1, R1, sp, mb, flag, 8, E, spec, spec_n, out, out_n, status,
                                      spec_ov=own, sum3=sum3, timeout_ns=2_000_000)
        s3 = sum3.cpu().tolist()
        assert s3[0] == -1 and s3[1] == 0 and s3[2] == int(own[0].item())
    finally:
        torch.cuda.synchronize()
        sc.xchg_free(mb)


def test_peer_rows_exchange_single_process():
    """seqcdc_xchg_put_rows / seqcdc_xchg_wait_rows (the step's second exchange
    over peer memory), three 'ranks' whose tables live in one local mailbox:
    every table receives every row, the wait returns the rows packed, and a
    step that never arrives times out (status 1) instead of hanging."""
    P, nw = 3, 3
    mb, _ = sc.xchg_alloc(4096)
    try:
        tables = torch.tensor([mb + 1024 * q for q in range(P)], dtype=torch.int64, device="cuda")
        rows = [torch.tensor([100 * r + 1, 100 * r + 2, 100 * r + 3], dtype=torch.int64, device="cuda")
                for r in range(P)]
        for r in range(P):
            sc.xchg_put_rows_into(rows[r], tables, r, 5)
        for q in range(P):
            out = torch.full((P * nw,), -7, dtype=torch.int64, device="cuda")
            status = torch.full((1,), -1, dtype=torch.int64, device="cuda")
            sc.xchg_wait_rows_into(mb + 1024 * q, nw, P, 5, status, out=out, timeout_ns=1_000_000_000)
            assert int(status.item()) == 0
            assert out.cpu().tolist() == [100 * r + i for r in range(P) for i in (1, 2, 3)]
        status = torch.full((1,), -1, dtype=torch.int64, device="cuda")
        out = torch.full((P * nw,), -7, dtype=torch.int64, device="cuda")
        sc.xchg_wait_rows_into(mb, nw, P, 6, status, out=out, timeout_ns=2_000_000)
        assert int(status.item()) == 1 and out.cpu().tolist() == [-7] * (P * nw)
    finally:
        torch.cuda.synchronize()
        sc.xchg_free(mb)
