#!/usr/bin/env python
"""Single-GPU timing of the pieces of one sharded step except the NCCL
exchanges: the speculative range pass on a 1 GiB shard (+ halo), and the
seam re-synchronisation from a true entry (device path), as rank r > 0 does."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2505_21194_b200 as sc  # noqa: E402
from paper_2505_21194_b200.dist import CudaRangeBackend, Shard  # noqa: E402

n_per = 1 << 30
p = sc.SeqParams.table1(4, 1)
lo = n_per                                   # rank 1 of a 1 GiB-per-rank stream
buf = torch.empty(n_per + (CudaRangeBackend.TAIL + 1) * p.max_size, dtype=torch.uint8, device="cuda")
synth.fill_device("markov", 2, lo, buf)
prev = torch.empty(p.max_size * 4, dtype=torch.uint8, device="cuda")   # rank 0's tail -> its overhang
synth.fill_device("markov", 2, lo - 2 * p.max_size, prev)
be = CudaRangeBackend(p)
shard = Shard(buf, n_per, lo)
# a plausible true entry: the first cut >= lo of a chain started before lo
full = sc.chunk(torch.cat([prev, buf[:1 << 20]]), p)
entry = int(full[(full >= 2 * p.max_size)][0].item()) + lo - 2 * p.max_size
d_entry = torch.tensor([entry], dtype=torch.int64, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
res = []
# the predecessor's tail block, as rank 0 would send it (its own range_chunk_tail)
be0 = CudaRangeBackend(p)
buf0 = torch.empty(n_per + (CudaRangeBackend.TAIL + 1) * p.max_size, dtype=torch.uint8, device="cuda")
synth.fill_device("markov", 2, 0, buf0)
prev = be0.spec_dev_tail(Shard(buf0, n_per, 0), last=False).extra["block"].clone()
for it in range(8):
    ev[0].record()
    spec = be.spec_dev_tail(shard, last=False)
    ev[1].record()
    cur = be.merge_dev(shard, prev, spec)
    ev[2].record()
    h = cur.extra["sum3"].cpu()
    ev[3].record()
    torch.cuda.synchronize()
    if it >= 3:
        res.append([ev[i].elapsed_time(ev[i + 1]) for i in range(3)])
m = [sum(r[i] for r in res) / len(res) for i in range(3)]
st = be.status.cpu().tolist()
print(json.dumps({"shard_bytes": n_per, "spec_with_tail_ms": round(m[0], 4), "merge_ms": round(m[1], 4),
                  "host_read_ms": round(m[2], 4), "merged_via_tail": st[0] == 1, "tail_cuts_used": st[1],
                  "prev_tail_n": int(prev[2].item()),
                  "note": "plus two NCCL all_gathers per step (not measurable on one GPU)"}))
