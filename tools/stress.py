#!/usr/bin/env python
"""Randomised parity stress (GPU box): random parameters, data kinds, sizes,
segment lengths, alignments, flags and call forms (single stream / batch),
every result compared with the oracle.  Prints one JSON summary line; exits 1
on the first mismatch (printing the case to reproduce it).

  python tools/stress.py [seconds] [seed]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2505_21194_b200 as sc  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 600.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
KINDS = ["uniform", "markov", "zeroheavy", "rampmix"]


def rand_params():
    L = int(rng.integers(2, 9))
    pairs = bool(rng.random() < 0.15)
    mn = int(rng.choice([L, L + 1, 64, 300, 1024, 2048, 4096, 8192]))
    mn = max(mn, L)
    mx = int(mn * rng.choice([1, 1.5, 2, 4, 8])) + int(rng.integers(0, 3))
    return oracle.Params(int(rng.integers(0, 2)), L, int(rng.integers(1, 120)), int(rng.choice([0, 1, 7, 64, 256, 511, 600])),
                         mn, mx, signed=bool(rng.random() < 0.15), pairs=pairs)


def sp(p):
    return sc.SeqParams(p.mode, p.seq_length, p.skip_trigger, p.skip_size, p.min_size, p.max_size,
                        (sc.FLAG_SIGNED if p.signed else 0) | (sc.FLAG_PAIRS if p.pairs else 0))


def data(n):
    k = rng.choice(KINDS + ["alphabet", "const"])
    if k == "alphabet":
        return rng.integers(0, int(rng.choice([2, 3, 5])), n).astype(np.uint8), "alphabet"
    if k == "const":
        return np.full(n, int(rng.integers(0, 256)), np.uint8), "const"
    return synth.fill_host(str(k), int(rng.integers(0, 1000)), int(rng.integers(0, 1 << 20)), n), str(k)


def range_draws(n, p):
    """The random draws range_case makes (so a replay can skip cases)."""
    P = int(rng.integers(2, 6))
    R = sorted(set([0, n] + rng.integers(p.max_size, n - p.max_size, P - 1).tolist()))
    return R


def range_case(b, n, p, R=None):
    """The multi-GPU seam protocol emulated in one process: P contiguous ranges
    (each with its halo), speculative pass + tail per range, then in rank order
    the local merge with the previous range's tail block (when that range's
    overhang stayed speculative) or a re-walk from the true entry."""
    E = 96
    if R is None:
        R = range_draws(n, p)
    R = [x for i, x in enumerate(R) if i == 0 or x - R[i - 1] >= p.max_size or x == n]
    if R[-1] != n:
        R.append(n)
    P = len(R) - 1
    q = sp(p)
    out, spec_ov, prev_blk, true_ov = [], None, None, None
    for r in range(P):
        lo, hi = R[r], R[r + 1]
        end = n if r == P - 1 else min(n, hi + (E + 1) * p.max_size)
        buf = torch.from_numpy(b[lo:end]).cuda()
        cap = sc.range_max_cuts(buf.numel(), hi - lo, q)
        spec = torch.empty(cap, dtype=torch.int64, device="cuda")
        spec_n = torch.zeros(1, dtype=torch.int64, device="cuda")
        blk = torch.zeros(3 + E, dtype=torch.int64, device="cuda")
        sc.range_chunk_tail_into(buf, hi - lo, lo, q, spec, spec_n, 0 if r == P - 1 else E, blk)
        if r == 0:
            cuts = spec[: int(spec_n.item())].cpu().numpy().astype(np.uint64)
            ov = int(blk[0].item())
        else:
            res = torch.empty(cap, dtype=torch.int64, device="cuda")
            res_n = torch.zeros(1, dtype=torch.int64, device="cuda")
            status = torch.zeros(4, dtype=torch.int64, device="cuda")
            if prev_spec_ov == true_ov:        # the previous tail continues the true chain
                sum3 = torch.zeros(3, dtype=torch.int64, device="cuda")
                sc.range_merge_tail_into(buf, hi - lo, lo, q, prev_blk, E, spec, spec_n, res, res_n, status,
                                         spec_ov=blk, sum3=sum3)
            else:
                sc.range_resync_into(buf, hi - lo, true_ov - lo, lo, q, spec, spec_n, res, res_n, status)
            cuts = res[: int(res_n.item())].cpu().numpy().astype(np.uint64)
            ov = int(status[3].item())
        out.append(cuts)
        prev_blk, prev_spec_ov, true_ov = blk, int(blk[0].item()), ov
    return np.concatenate(out) if out else np.zeros(0, np.uint64), oracle.chunk(b, p)


t0 = time.time()
start = int(os.environ.get("STRESS_START", "0"))      # replay: skip (draw only) the cases before it
only = os.environ.get("STRESS_ONLY") is not None       # ... and stop after that one
cases = cuts_checked = 0
forms = {"single": 0, "batch": 0, "range": 0}
while time.time() - t0 < budget:
    p = rand_params()
    n = int(rng.choice([0, 1, 5, 100, 4096, 100000, 1 << 20, 5 << 20, 24 << 20])) + int(rng.integers(0, 4096))
    b, kind = data(n)
    G = int(rng.choice([0, 0, 1 << 14, 1 << 16, 1 << 18]))
    sc.set_segment_bytes(G)
    u = rng.random()
    form = "batch" if u < 0.25 else ("range" if u < 0.45 and n >= 8 * p.max_size else "single")
    if cases < start:                            # consume exactly the draws the case would make
        if form == "range":
            range_draws(n, p)
        elif form == "single":
            rng.integers(0, 16)
        else:
            ns = int(rng.integers(1, 12))
            if ns > 1:
                rng.integers(0, n + 1, ns - 1)
        sc.set_segment_bytes(0)
        cases += 1
        continue
    if only and cases > start:
        break
    if os.environ.get("STRESS_DRY"):            # replay aid: leave the case for the caller
        CASE = {"b": b, "n": n, "p": p, "kind": kind, "G": G, "form": form,
                "R": range_draws(n, p) if form == "range" else None}
        break
    if os.environ.get("STRESS_LOG"):           # the case about to run (survives a crash)
        with open(os.environ["STRESS_LOG"], "a") as f:
            f.write(json.dumps({"case": cases, "form": form, "kind": kind, "n": n, "G": G, "params": repr(p)}) + "\n")
    try:
        if form == "range":
            got, want = range_case(b, n, p)
        elif form == "single":
            off = int(rng.integers(0, 16))
            buf = torch.zeros(n + off, dtype=torch.uint8, device="cuda")
            if n:
                buf[off:] = torch.from_numpy(b).cuda()
            got = sc.chunk(buf[off:], sp(p)).cpu().numpy().astype(np.uint64)
            want = oracle.chunk(b, p)
        else:
            ns = int(rng.integers(1, 12))
            cutsp = np.sort(rng.integers(0, n + 1, ns - 1)) if ns > 1 else np.zeros(0, np.int64)
            offs = np.concatenate([[0], cutsp, [n]]).astype(np.uint64)
            gc, gi = sc.chunk_batch(torch.from_numpy(b).cuda() if n else torch.zeros(0, dtype=torch.uint8, device="cuda"),
                                    torch.from_numpy(offs.astype(np.int64)).cuda(), sp(p))
            got = np.concatenate([gi.cpu().numpy().astype(np.uint64), gc.cpu().numpy().astype(np.uint64)])
            wc, wi = oracle.chunk_batch(b, offs, p)
            want = np.concatenate([wi.astype(np.uint64), wc.astype(np.uint64)])
    finally:
        sc.set_segment_bytes(0)
    cases += 1
    forms[form] += 1
    cuts_checked += int(want.size)
    if got.shape != want.shape or not np.array_equal(got, want):
        print(json.dumps({"mismatch": True, "form": form, "kind": kind, "n": n, "G": G, "params": repr(p)}))
        sys.exit(1)
if os.environ.get("STRESS_DRY"):
    sys.exit(0) if __name__ == "__main__" else None
print(json.dumps({"stress": "ok", "cases": cases, "forms": forms, "cuts_checked": cuts_checked,
                  "seconds": round(time.time() - t0, 1), "walker": os.environ.get("SEQCDC_WALKER", "auto")}))
