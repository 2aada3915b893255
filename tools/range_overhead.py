#!/usr/bin/env python
"""Single-GPU timing of the pieces of one sharded step (everything but the
exchanges between GPUs), on rank 1's shard of a config-5-shaped stream:

  python tools/range_overhead.py [SHARD_GIB ...]      (default 8 16 32)

plain   = seqcdc_chunk on the shard's bytes (what one GPU would do alone)
spec    = seqcdc_range_chunk_tail (speculative chain + the tail past the overhang)
merge   = seqcdc_range_merge_tail with rank 0's real block (local merge)
read    = the step's one host read (the summary row)
One JSON line per shard size."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2505_21194_b200 as sc  # noqa: E402
from paper_2505_21194_b200.dist import CudaRangeBackend, Shard  # noqa: E402

GiB = 1 << 30
p = sc.SeqParams.table1(8, 0)
halo = (CudaRangeBackend.TAIL + 1) * p.max_size


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(reps):
        fn()
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / reps


for gib in [int(x) for x in sys.argv[1:]] or [8, 16, 32]:
    n_per = gib * GiB
    buf0 = torch.empty(n_per + halo, dtype=torch.uint8, device="cuda")
    synth.fill_device("rampmix", 5, 0, buf0)
    buf1 = torch.empty(n_per + halo, dtype=torch.uint8, device="cuda")
    synth.fill_device("rampmix", 5, n_per, buf1)
    be0, be1 = CudaRangeBackend(p), CudaRangeBackend(p)
    sh0, sh1 = Shard(buf0, n_per, 0), Shard(buf1, n_per, n_per)
    block0 = be0.spec_dev_tail(sh0, last=False).extra["block"].clone()
    torch.cuda.synchronize()
    plain_cuts = torch.empty(sc.max_cuts(n_per, p), dtype=torch.int64, device="cuda")
    plain_n = torch.zeros(1, dtype=torch.int64, device="cuda")
    ws = torch.empty(sc.workspace_size(n_per, 1, p), dtype=torch.uint8, device="cuda")
    t_plain = timed(lambda: sc.chunk_into(buf1[:n_per], p, plain_cuts, plain_n, workspace=ws))
    walker = sc.build_info().split(";")[1].strip()
    del ws
    spec = be1.spec_dev_tail(sh1, last=False)
    t_spec = timed(lambda: be1.spec_dev_tail(sh1, last=False))
    t_merge = timed(lambda: be1.merge_dev(sh1, block0, spec))
    cur = be1.merge_dev(sh1, block0, spec)
    t_read = timed(lambda: cur.extra["sum3"].cpu())
    st = be1.status.cpu().tolist()
    print(json.dumps({"shard_GiB": gib, "walker": walker, "plain_ms": round(t_plain, 4),
                      "spec_with_tail_ms": round(t_spec, 4), "merge_ms": round(t_merge, 4),
                      "host_read_ms": round(t_read, 4),
                      "step_over_plain": round((t_spec + t_merge + t_read) / t_plain, 4),
                      "merged_via_tail": st[0] == 1, "tail_n": int(be1.block[2].item()) if False else int(block0[2].item()),
                      "note": "plus the two exchanges between GPUs (peer stores or all_gathers), not measurable here"}),
          flush=True)
    del buf0, buf1, be0, be1, plain_cuts
    torch.cuda.empty_cache()
