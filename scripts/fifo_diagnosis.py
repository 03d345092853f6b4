#!/usr/bin/env python
"""Why the paper's FIFO + stickiness scheme thrashes under INDEPENDENT random
per-rank orders, from the device trace.

Workload: C3 (64 mixed collectives, 8 ranks), every rank in its own random
permutation, all SQEs pre-enqueued, one daemon launch, tracing on.  For each
daemon block index b the same collective lane runs on block b of every rank
(a collective's lanes start at block collId mod G on all ranks), so the ranks
can only make progress together when their block b runs the same collective
at the same time.  From the per-block traces we compute:

* qlen_at_first_progress: task-queue length (admitted, not completed) of a
  block when it commits its first slice -- under FIFO the queue grows by one
  SQE only when every queued entry is stalled, so a block must
  admit entries until the ranks' admitted sets intersect;
* the same quantity predicted by a plain model: the smallest k such that the
  first k entries of the 8 permutations share a collective (Monte Carlo over
  the SAME seeded orders);
* aligned_frac: fraction of the launch during which ALL ranks' block b run the
  same collective (gang-scheduled), and pair_frac: fraction during which a
  rank and its upstream run the same collective (a ring edge can move data);
* runs per committed slice, median run length, preemptions.

The same statistics for the consistent order (every rank ascending) and for
the priority policy are printed beside it.
"""
import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from inputs import workloads  # noqa: E402
from paper_2303_06324_b200 import harness, occl  # noqa: E402


def intervals(tr):
    """[(t0, t1, coll)] of collective runs on one block (switch_in -> done/preempt)."""
    out, cur = [], None
    for t, ev, c, a in tr:
        if ev == "switch_in":
            cur = (t, c)
        elif ev in ("done", "preempt") and cur is not None:
            out.append((cur[0], t, cur[1]))
            cur = None
    return out


def coverage(ivs_by_rank, t_lo, t_hi, pair=False):
    """Time during which all ranks (or rank r and r-1) run the same collective, and
    the start of the first all-rank alignment (None if never)."""
    n = len(ivs_by_rank)
    edges = sorted({t for ivs in ivs_by_rank for (a, b, _) in ivs for t in (a, b)} | {t_lo, t_hi})
    idx = [0] * n
    aligned, paired, first = 0, 0, None
    for k in range(len(edges) - 1):
        a, b = edges[k], edges[k + 1]
        mid = (a + b) / 2
        cur = []
        for r in range(n):
            ivs = ivs_by_rank[r]
            while idx[r] < len(ivs) and ivs[idx[r]][1] <= mid:
                idx[r] += 1
            i = idx[r]
            cur.append(ivs[i][2] if i < len(ivs) and ivs[i][0] <= mid < ivs[i][1] else None)
        if cur[0] is not None and all(c == cur[0] for c in cur):
            aligned += b - a
            if first is None:
                first = a
        paired += (b - a) * sum(1 for r in range(n) if cur[r] is not None and cur[r] == cur[r - 1]) / n
    return aligned, paired, first


def predicted_intersection(orders, lanes_of):
    """Smallest k such that the first k admitted entries of every rank share a collective
    (only collectives with a lane on this block count)."""
    n = len(orders)
    seqs = [[c for c in o if lanes_of(c)] for o in orders]
    m = min(len(s) for s in seqs)
    for k in range(1, m + 1):
        common = set(seqs[0][:k])
        for s in seqs[1:]:
            common &= set(s[:k])
        if common:
            return k
    return None


def run(policy, stick, order_kind, seed, args):
    n, G = 8, args.grid
    comms = harness.ring(n, 0, gridBlocks=G, maxColl=256, autoLaunch=0, orderPolicy=policy, stickiness=stick,
                         traceCap=1 << 16)
    try:
        colls, orders = workloads.c3(n, 64, seed)
        if order_kind == "consistent":
            orders = [list(range(len(colls)))] * n
        bufs = {c.coll_id: harness.buffers(c.kind, c.dtype, n, c.count, comms) for c in colls}
        jobs = [(c.coll_id, c.kind, c.dtype, c.count, c.root, bufs[c.coll_id]) for c in colls]
        torch.cuda.synchronize()
        for c in comms:
            c.trace_reset()
        before = [c.stats() for c in comms]
        ms = harness.timed_batch(comms, jobs, orders, timeout_s=600)
        pre = sum(c.stats()["preemptions"] - b["preemptions"] for c, b in zip(comms, before))
        blocks = {}
        nblocks = {c.coll_id: comms[0].coll_blocks(c.kind, c.count, c.dtype) for c in colls}   # occlCollBlocks
        q_first, q_pred, aligned_f, pair_f, runs_per_slice, run_len = [], [], [], [], [], []
        q_align, t_align = [], []
        for b in range(0, G, max(1, G // args.sample_blocks)):
            trs = [comms[r].trace(b) for r in range(n)]
            if not all(trs):
                continue
            t_lo = min(tr[0][0] for tr in trs)
            t_hi = max(tr[-1][0] for tr in trs)
            ivs = [intervals(tr) for tr in trs]
            al, pa, t_first = coverage(ivs, t_lo, t_hi)
            if t_first is not None:
                # queue length (admitted, not completed) of every rank's block b at the
                # first moment all ranks ran the same collective
                for r in range(n):
                    f = sum(1 for t, ev, c, a in trs[r] if ev == "fetch" and t <= t_first)
                    d = sum(1 for t, ev, c, a in trs[r] if ev == "done" and t <= t_first)
                    q_align.append(f - d)
                t_align.append((t_first - t_lo) / 1e3)
            aligned_f.append(al / max(1, t_hi - t_lo))
            pair_f.append(pa / max(1, t_hi - t_lo))
            for r in range(n):
                fetched, done, first = 0, 0, None
                nrun = len(ivs[r])
                nsl = sum(1 for t, ev, c, a in trs[r] if ev == "issue")
                runs_per_slice.append(nrun / max(1, nsl))
                run_len.extend((t1 - t0) / 1e3 for t0, t1, _ in ivs[r])
                for t, ev, c, a in trs[r]:
                    if ev == "fetch":
                        fetched += 1
                    elif ev == "done":
                        done += 1
                    elif ev == "issue" and first is None:
                        first = fetched - done
                if first is not None:
                    q_first.append(first)
            # the plain model: FIFO admits in submission order; collectives whose
            # lane set covers block b are the ones this block admits
            lanes = (lambda c, b=b: (b - c % G) % G < nblocks[c])
            q_pred.append(predicted_intersection(orders, lanes))
        res = {"policy": ["fifo", "priority"][policy], "stickiness": stick, "order": order_kind, "seed": seed,
               "ms": ms, "preemptions": pre,
               "qlen_at_first_progress_median": statistics.median(q_first) if q_first else None,
               "qlen_at_first_alignment_median": statistics.median(q_align) if q_align else None,
               "us_to_first_alignment_median": statistics.median(t_align) if t_align else None,
               "qlen_predicted_intersection_median": statistics.median([q for q in q_pred if q]) if any(q_pred) else None,
               "aligned_frac_median": float(np.median(aligned_f)) if aligned_f else None,
               "pair_frac_median": float(np.median(pair_f)) if pair_f else None,
               "runs_per_slice_median": float(np.median(runs_per_slice)) if runs_per_slice else None,
               "run_us_median": float(np.median(run_len)) if run_len else None}
        return res
    finally:
        occl.destroy_group(comms)
        torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", type=int, default=2)
    ap.add_argument("--grid", type=int, default=18)
    ap.add_argument("--sample-blocks", type=int, default=6)
    ap.add_argument("--out", default="gpurun_out/fifo_diagnosis.jsonl")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    with open(args.out, "w") as f:
        for seed in range(args.seeds):
            for policy, stick, ok in ((0, 1, "consistent"), (0, 1, "random"), (0, 0, "random"), (1, 1, "random")):
                r = run(policy, stick, ok, seed, args)
                print(json.dumps(r), flush=True)
                f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
