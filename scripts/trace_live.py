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
    ap.add_argument("--gap-us", type=float, default=0.0, help="Exp-distributed gaps between submissions")
    ap.add_argument("--per-coll", action="store_true", help="per-collective device timing of every run")
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
    dur = {}
    if a.per_coll:                                     # standalone device time of each collective
        for k, job in enumerate(jobs):
            dur[job[0]] = sorted(harness.timed_batch(comms, [job]) for _ in range(3))[1]
        for c in comms:
            c.set_auto_launch(True)
    runs = []
    worst = None
    try:
        for it in range(a.runs):
            comms[0].quiesce(10)                       # the event-driven daemon quit after the last run
            for c in comms:
                c.trace_reset()
            before = [c.stats() for c in comms]
            if a.gap_us:
                delays = workloads.arrival_delays(n, len(colls), a.gap_us * 1e-6, it)
            r = harness.live_run(comms, jobs, orders, delays, timeout_s=120)
            st = {k: sum(c.stats()[k] - b[k] for c, b in zip(comms, before))
                  for k in ("launches", "quits", "preemptions", "exits", "sqeFetched")}
            row = {"run": it, "makespan_ms": r["makespan_ms"], **st}
            if a.per_coll:
                comms[0].quiesce(10)
                pc = {}
                for k, job in enumerate(jobs):
                    cid = job[0]
                    fet, sw, dn = [], [], []
                    for rk in range(n):
                        tr = comms[rk].trace(cid % 18)
                        f = [t for t, e, c, x in tr if e == "fetch" and c == cid]
                        if not f:
                            continue
                        fet.append(f[-1])
                        s_ = [t for t, e, c, x in tr if e == "switch_in" and c == cid and t >= f[-1]]
                        d_ = [t for t, e, c, x in tr if e == "done" and c == cid and t >= f[-1]]
                        if s_:
                            sw.append(s_[0])
                        if d_:
                            dn.append(d_[-1])
                    if len(fet) == n and len(sw) == n and len(dn) == n:
                        pc[cid] = {"ready_host_ms": r["ready_ms"][0][k], "last_fetch_to_last_switch_us": (max(sw) - max(fet)) / 1e3,
                                   "last_switch_to_last_done_us": (max(dn) - max(sw)) / 1e3,
                                   "first_switch_to_last_done_us": (max(dn) - min(sw)) / 1e3,
                                   "standalone_us": dur[cid] * 1e3}
                t0 = None
                row["per_coll"] = pc
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
