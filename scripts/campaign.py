#!/usr/bin/env python
"""Deadlock campaign at 8 ranks where preemption actually happens (VERDICT r01
next #2; BASELINE north star: 0 deadlocks across 10,000 random per-rank
submission orders; PAPER.md:736-739 the misordered-collectives demo).

Each trial: 8 all-reduces of 256 B .. 1 MiB (log-uniform) with an
independent random permutation per rank (inputs.workloads.deadlock_trial),
int32 inputs, a 10 s per-trial watchdog, and EVERY output checked against the
order-free closed form (the wrapped int32 sum, computed with torch on the
inputs).  Two campaigns:

* fifo  : the paper's policy -- FIFO task queues + stickiness,
          all SQEs pre-enqueued, one daemon launch per trial; misordered heads
          force spin -> preempt -> save -> resume;
* live  : the priority policy with LIVE arrival -- per-rank submitter threads
          feed the running event-driven daemon after a barrier, each rank with
          its own order and Exp(mean) gaps (harness.live_run), so a rank's queue
          front changes while collectives run and blocked collectives yield.

Reported: trials, timeouts, mismatches, total preemptions and the number of
trials in which at least one preemption happened, wall time.
"""
import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from inputs import workloads  # noqa: E402
from paper_2303_06324_b200 import harness, occl  # noqa: E402

MAXC = (1 << 20) // 4


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", choices=["fifo", "live"], required=True)
    ap.add_argument("--trials", type=int, default=10000)
    ap.add_argument("--seed0", type=int, default=0)
    ap.add_argument("--gap-us", type=float, default=30.0, help="live: mean Exp gap between submissions")
    ap.add_argument("--out", default="gpurun_out/campaign")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    n, k = 8, 8
    cfg = dict(gridBlocks=4, maxColl=16, sliceBytes=16384, minBlockBytes=65536, spinBase=256, spinStep=32,
               spinMin=16)
    if a.mode == "fifo":
        comms = harness.ring(n, 0, autoLaunch=0, orderPolicy=0, stickiness=1, **cfg)
    else:
        comms = harness.ring(n, 0, autoLaunch=1, orderPolicy=1, stickiness=1, quitIdleNs=500_000, **cfg)
    g = torch.Generator(device="cuda")
    g.manual_seed(a.seed0)
    send = [[torch.empty(MAXC, dtype=torch.int32, device=0) for _ in range(n)] for _ in range(k)]
    recv = [[torch.empty(MAXC, dtype=torch.int32, device=0) for _ in range(n)] for _ in range(k)]
    timeouts = mismatches = 0
    pre_total = trials_pre = 0
    per_trial = []
    t0 = time.time()
    try:
        for trial in range(a.trials):
            seed = a.seed0 + trial
            colls, orders = workloads.deadlock_trial(n, k, seed=seed)
            jobs = []
            for c in colls:
                for r in range(n):
                    send[c.coll_id][r][:c.count] = torch.randint(-2**31, 2**31 - 1, (c.count,), dtype=torch.int32,
                                                                 device=0, generator=g)
                    recv[c.coll_id][r][:c.count].fill_(0)
                bufs = [(send[c.coll_id][r][:c.count], recv[c.coll_id][r][:c.count]) for r in range(n)]
                jobs.append((c.coll_id, "allreduce", "i32", c.count, 0, bufs))
            torch.cuda.synchronize()
            before = sum(c.stats()["preemptions"] for c in comms)
            try:
                if a.mode == "fifo":
                    harness.timed_batch(comms, jobs, orders, timeout_s=10.0)
                else:
                    delays = workloads.arrival_delays(n, k, a.gap_us * 1e-6, seed)
                    harness.live_run(comms, jobs, orders, delays, timeout_s=10.0)
            except (occl.OcclError, TimeoutError) as e:
                timeouts += 1
                print(f"trial {trial}: {e!r}", flush=True)
                break
            pre = sum(c.stats()["preemptions"] for c in comms) - before
            pre_total += pre
            trials_pre += pre > 0
            per_trial.append(pre)
            for cid, kind, dt, count, root, bufs in jobs:
                acc = bufs[0][0].clone()
                for s, _ in bufs[1:]:
                    acc = acc + s                      # torch int32 addition wraps (two's complement)
                if not all(torch.equal(r, acc) for _, r in bufs):
                    mismatches += 1
            if trial % 1000 == 999:
                print(f"{a.mode}: {trial + 1} trials, {timeouts} timeouts, {mismatches} mismatches, "
                      f"{pre_total} preemptions, {trials_pre} trials with preemptions, {time.time() - t0:.0f} s",
                      flush=True)
    finally:
        occl.destroy_group(comms)
    per_trial.sort()
    res = {"mode": a.mode, "trials": len(per_trial), "requested": a.trials, "timeouts": timeouts,
           "mismatches": mismatches, "preemptions": pre_total, "trials_with_preemption": trials_pre,
           "preemptions_per_trial_median": per_trial[len(per_trial) // 2] if per_trial else None,
           "preemptions_per_trial_max": per_trial[-1] if per_trial else None,
           "wall_s": time.time() - t0, "config": cfg, "gap_us": a.gap_us if a.mode == "live" else None}
    print("RESULT", json.dumps(res), flush=True)
    with open(a.out + f"_{a.mode}.json", "w") as f:
        json.dump(res, f, indent=1)
    return 0 if timeouts == 0 and mismatches == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
