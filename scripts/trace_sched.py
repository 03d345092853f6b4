"""Scheduler timeline from the device trace: C3 (64 mixed collectives, 8 ranks) in
one consistent order under the FIFO and priority policies.  Per block: busy time
inside collective runs, gaps between runs (scheduling: SQ fetch, admission,
context load), number of switch-ins, first-run start."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from inputs import workloads  # noqa: E402
from paper_2303_06324_b200 import harness, occl  # noqa: E402


def main():
    n = 8
    out = {}
    for policy in (0, 1):
        comms = harness.ring(n, 0, gridBlocks=18, maxColl=256, autoLaunch=0, orderPolicy=policy, traceCap=1 << 15)
        colls, orders = workloads.c3(n, 64, 0)
        bufs = {c.coll_id: harness.buffers(c.kind, c.dtype, n, c.count, comms) for c in colls}
        jobs = [(c.coll_id, c.kind, c.dtype, c.count, c.root, bufs[c.coll_id]) for c in colls]
        consistent = [sorted(range(len(colls)))] * n
        harness.timed_batch(comms, jobs, consistent)
        for c in comms:
            c.trace_reset()
        ms = harness.timed_batch(comms, jobs, consistent)
        busy, gaps, nsw, first, fetch_span = [], [], [], [], []
        t0 = None
        for r in range(n):
            for b in range(18):
                tr = comms[r].trace(b)
                if not tr:
                    continue
                t0 = tr[0][0] if t0 is None else min(t0, tr[0][0])
        for r in range(n):
            for b in range(18):
                tr = comms[r].trace(b)
                last_end, bsy, gp, sw = None, 0, 0, 0
                cur = None
                fetches = [t for t, ev, c, a in tr if ev == "fetch"]
                if fetches:
                    fetch_span.append((fetches[-1] - fetches[0]) / 1e3)
                for t, ev, c, a in tr:
                    if ev == "switch_in":
                        sw += 1
                        if last_end is not None:
                            gp += t - last_end
                        else:
                            first.append((t - t0) / 1e3)
                        cur = t
                    elif ev in ("done", "preempt") and cur is not None:
                        bsy += t - cur
                        last_end = t
                        cur = None
                busy.append(bsy / 1e3)
                gaps.append(gp / 1e3)
                nsw.append(sw)
        out[["fifo", "priority"][policy]] = {
            "ms": ms, "busy_us_median": float(np.median(busy)), "gap_us_median": float(np.median(gaps)),
            "gap_us_max": float(np.max(gaps)), "switch_ins_median": float(np.median(nsw)),
            "first_run_us_median": float(np.median(first)), "first_run_us_max": float(np.max(first)),
            "fetch_span_us_median": float(np.median(fetch_span)) if fetch_span else None}
        print(json.dumps({["fifo", "priority"][policy]: out[["fifo", "priority"][policy]]}), flush=True)
        occl.destroy_group(comms)
        del bufs
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
