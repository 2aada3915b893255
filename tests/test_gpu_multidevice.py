"""Two devices driven from one process: the library keeps its SM counts,
occupancies, function attributes and memory pool per device, and the binding
runs each call with the data's device current.  Skipped with fewer than two
GPUs (the pool's boxes have one; the driver's 8-GPU runs have eight)."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2505_21194_b200 as sc  # noqa: E402


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_calls_alternate_between_devices():
    p = oracle.table1(8)
    sp = sc.SeqParams(p.mode, p.seq_length, p.skip_trigger, p.skip_size, p.min_size, p.max_size)
    b = synth.fill_host("rampmix", 61, 0, 24 << 20)
    want = oracle.chunk(b, p)
    torch.cuda.set_device(0)
    for dev in (1, 0, 1):                     # device 1's first call with device 0 current
        d = torch.from_numpy(b).to(f"cuda:{dev}")
        got = sc.chunk(d, sp).cpu().numpy().astype(np.uint64)
        assert np.array_equal(got, want), dev
    # a batch on device 1 (k_stitch's dynamic shared memory attribute is per device)
    allb, offs = synth.batch_host(5, 12, 1 << 20)
    cuts, idx = sc.chunk_batch(torch.from_numpy(allb).to("cuda:1"), torch.from_numpy(offs.astype(np.int64)).to("cuda:1"), sp)
    wc, wi = oracle.chunk_batch(allb, offs, p)
    assert np.array_equal(cuts.cpu().numpy().astype(np.uint64), wc)


def test_binding_refuses_undersized_outputs():
    """The C ABI takes no capacities: the binding checks them (and dtypes)."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    p = sc.SeqParams.table1(8)
    d = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
    small = torch.empty(sc.max_cuts(d.numel(), p) - 1, dtype=torch.int64, device="cuda")
    n = torch.zeros(1, dtype=torch.int64, device="cuda")
    with pytest.raises(sc.SeqCDCError):
        sc.chunk_into(d, p, small, n)
    with pytest.raises(sc.SeqCDCError):
        sc.chunk_into(d, p, torch.empty(sc.max_cuts(d.numel(), p), dtype=torch.int32, device="cuda"), n)
