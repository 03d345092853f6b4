#!/usr/bin/env python
"""Timeline of LIVE runs (per-rank submitter threads, event-driven daemon) from
the device trace: which runs are slow and why (quit / relaunch churn, waiting
for SQEs, preemptions).  Workload: ResNet-50 25 MiB buckets (C4), 8 virtual
ranks, consistent order, no jitter, repeated --runs times; per run: makespan,
daemon launches, quits, preemptions, and for the slowest run a per-rank event
summary of block 0 (start / fetch / switch-in / preempt / done / quit / exit
with times relative to the run's first device event)."""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from inputs import workloads  # noqa: E402
from paper_2303_06324_b200 import harness, occl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--runs", type=int, default=20)
    ap.add_argument("--policy", type=int, default=1)
    ap.add_argument("--workload", default="resnet50")
    ap.add_argument("--quit-idle-ns", type=int, default=0)
    ap.add_argument("--out", default="gpurun_out/trace_live.json")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    n = 8
    extra = {"quitIdleNs": a.quit_idle_ns} if a.quit_idle_ns else {}
    comms = harness.ring(n, 0, gridBlocks=18, maxColl=256, orderPolicy=a.policy, traceCap=1 << 14, **extra)
    colls, _ = workloads.c4(a.workload, n, 0)
    bufs = {c.coll_id: harness.buffers(c.kind, c.dtype, n, c.count, comms) for c in colls}
    jobs = [(c.coll_id, c.kind, c.dtype, c.count, c.root, bufs[c.coll_id]) for c in colls]
    orders = [list(range(len(colls)))] * n
    delays = [[0.0] * len(colls)] * n
    runs = []
    worst = None
    try:
        for it in range(a.runs):
            comms[0].quiesce(10)                       # the event-driven daemon quit after the last run
            for c in comms:
                c.trace_reset()
            before = [c.stats() for c in comms]
            r = harness.live_run(comms, jobs, orders, delays, timeout_s=120)
            st = {k: sum(c.stats()[k] - b[k] for c, b in zip(comms, before))
                  for k in ("launches", "quits", "preemptions", "exits", "sqeFetched")}
            row = {"run": it, "makespan_ms": r["makespan_ms"], **st}
            runs.append(row)
            print(json.dumps(row), flush=True)
            if worst is None or r["makespan_ms"] > worst[0]:
                comms[0].quiesce(10)
                evs = {}
                for rk in range(n):
                    for b in range(18):
                        evs[(rk, b)] = [e for e in comms[rk].trace(b) if e[1] not in ("issue", "sdone", "publish")]
                worst = (r["makespan_ms"], it, evs)
        ms, it, evs = worst
        t0 = min(e[0][0] for e in evs.values() if e)
        summary = {f"{rk}.{b}": [(round((t - t0) / 1e3, 2), ev, c, x) for t, ev, c, x in tr]
                   for (rk, b), tr in evs.items()}
        out = {"runs": runs, "worst_run": it, "worst_ms": ms, "events_us": summary}
        with open(a.out, "w") as f:
            json.dump(out, f)
        print(json.dumps({"worst_run": it, "worst_ms": ms}))
    finally:
        occl.destroy_group(comms)


if __name__ == "__main__":
    main()
