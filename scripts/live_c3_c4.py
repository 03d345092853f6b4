#!/usr/bin/env python
"""C3 / C4 with asynchronous, jittered arrival into a LIVE daemon (VERDICT r01
next #2; BASELINE.json configs[2], configs[3]).

For every (workload, policy variant, seed, repeat):
  * consistent: every rank submits in the SAME order (ascending collId, i.e.
    priority order), with its own Exp(mean) gaps between submissions;
  * random    : every rank submits in its OWN random permutation, same gap law.
Per-rank submitter threads (paper_2303_06324_b200.harness.live_run) start after
a barrier and feed the event-driven daemon (autoLaunch = 1, voluntary quit on).
C3 = one round of 64 mixed collectives (1-64 MiB); C4 = `iterations` DP steps
of gradient buckets, ids resubmitted each step.  mean gap = one collective's
time (measured: consistent no-jitter makespan / #collectives).

Reported per row: makespan (C3) or median iteration time (C4), preemption
counts, overhead = T_random / T_consistent - 1, and -- because a collective
cannot start before its LAST rank submitted it, which under independent random
orders is late in the submission window whatever the scheduler does -- the
overhead against the ideal gang-scheduled makespan for the SAME arrivals
(ideal_ms: the collectives back to back in the order they became ready, each
at its standalone device time; DESIGN.md §5 "live arrival").  A summary per
(workload, variant) gives the median and min-max over seeds x repeats.
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from inputs import workloads  # noqa: E402
from paper_2303_06324_b200 import harness, occl  # noqa: E402

VARIANTS = {"priority": (1, 1), "fifo+stickiness": (0, 1), "fifo-constT": (0, 0)}


def workload(name, n, seed):
    if name == "c3":
        return workloads.c3(n, 64, seed)
    if name == "resnet50-buckets":
        return workloads.c4("resnet50", n, seed)
    if name == "resnet50-tensors":
        return workloads.c4("resnet50", n, seed, per_tensor=True)
    if name == "bert-large-buckets":
        return workloads.c4("bert-large", n, seed)
    raise ValueError(name)


def stats_delta(comms, before):
    after = [c.stats() for c in comms]
    return {k: sum(a[k] - b[k] for a, b in zip(after, before)) for k in ("preemptions", "ctxSaves", "quits",
                                                                        "launches", "cqeWritten")}


def ideal_ms(ready, dur):
    """Ideal gang-scheduled makespan given the arrivals: the collectives run one
    after another, each as soon as every rank submitted it (ready[k], ms after the
    iteration's first submission) and the previous one finished, each taking its
    standalone device time dur[k] -- what a scheduler with perfect knowledge of
    the arrivals achieves without preemption cost (collectives using fewer blocks
    could overlap, so this is a reference, not a strict bound)."""
    t = 0.0
    for k in sorted(ready, key=lambda j: ready[j]):
        t = max(t, ready[k]) + dur[k]
    return t


def standalone_ms(comms, jobs):
    """Device time of each collective alone (one daemon launch each, median of 3)."""
    out = {}
    for k, job in enumerate(jobs):
        ts = sorted(harness.timed_batch(comms, [job]) for _ in range(3))
        out[k] = ts[1]
    return out


def one(comms, jobs, n, ncoll, iters, seed, rep, mean_gap, order_kind):
    base = seed * 7919 + rep * 104729 + (0 if order_kind == "consistent" else 1)
    if order_kind == "consistent":
        of = lambda it: [list(range(ncoll))] * n
    else:
        of = lambda it: workloads.iteration_orders(n, ncoll, base, it)
    df = lambda it: workloads.arrival_delays(n, ncoll, mean_gap, base * 1009 + it)
    before = [c.stats() for c in comms]
    r = harness.live_run(comms, jobs, None, None, iterations=iters, orders_fn=of, delays_fn=df, timeout_s=600)
    st = stats_delta(comms, before)
    t = r["makespan_ms"] if iters == 1 else statistics.median(r["iter_ms"])
    return t, st, r


def ideal_of(r, dur, iters):
    v = [ideal_ms(rd, dur) for rd in r["ready_ms"]]
    return v[0] if iters == 1 else statistics.median(v)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ranks", type=int, default=8)
    ap.add_argument("--seeds", type=int, default=10)
    ap.add_argument("--repeats", type=int, default=3)
    ap.add_argument("--workloads", default="c3,resnet50-buckets,resnet50-tensors,bert-large-buckets")
    ap.add_argument("--variants", default="priority,fifo+stickiness,fifo-constT")
    ap.add_argument("--iterations", type=int, default=200, help="C4 DP iterations (priority variant)")
    ap.add_argument("--fifo-iterations", type=int, default=10, help="C4 iterations for FIFO variants")
    ap.add_argument("--fifo-seeds", type=int, default=3)
    ap.add_argument("--out", default="gpurun_out/live_c3_c4")
    ap.add_argument("--grid", type=int, default=18)
    ap.add_argument("--spin-ns", type=int, default=0)
    ap.add_argument("--stall-ns", type=int, default=-1)
    ap.add_argument("--spin-base", type=int, default=0)
    ap.add_argument("--spin-step", type=int, default=-1)
    ap.add_argument("--spin-min", type=int, default=0)
    ap.add_argument("--spin-cap", type=int, default=0)
    ap.add_argument("--quit-idle-ns", type=int, default=0)
    ap.add_argument("--ready-first", type=int, default=-1, help="-1: library default")
    ap.add_argument("--c3-gap", choices=["op", "zero"], default="op",
                    help="C3 inter-submission gap: Exp(one op) or back-to-back (SURVEY §8(d) C3)")
    ap.add_argument("--tag", default="")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    n = args.ranks
    rows = []
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    fout = open(args.out + ".jsonl", "w")
    for wname in args.workloads.split(","):
        for vname in args.variants.split(","):
            policy, stick = VARIANTS[vname]
            extra = {"spinNs": args.spin_ns} if args.spin_ns else {}
            if args.stall_ns >= 0:
                extra["stallNs"] = args.stall_ns
            for k, v in (("spinBase", args.spin_base), ("spinMin", args.spin_min), ("spinCap", args.spin_cap),
                         ("quitIdleNs", args.quit_idle_ns)):
                if v:
                    extra[k] = v
            if args.spin_step >= 0:
                extra["spinStep"] = args.spin_step
            if args.ready_first >= 0:
                extra["readyFirst"] = args.ready_first
            comms = harness.ring(n, 0, gridBlocks=args.grid, maxColl=256, orderPolicy=policy, stickiness=stick,
                                 **extra)
            fifo = policy == 0
            nseeds = min(args.seeds, args.fifo_seeds) if fifo else args.seeds
            for seed in range(nseeds):
                colls, _ = workload(wname, n, seed)
                ncoll = len(colls)
                iters = 1 if wname == "c3" else (args.fifo_iterations if fifo else args.iterations)
                bufs = {c.coll_id: harness.buffers(c.kind, c.dtype, n, c.count, comms) for c in colls}
                jobs = [(c.coll_id, c.kind, c.dtype, c.count, c.root, bufs[c.coll_id]) for c in colls]
                dur = standalone_ms(comms, jobs)
                for c in comms:
                    c.set_auto_launch(True)
                # calibration: consistent order, no jitter (also first touch of buffers / arena)
                t_cal, _, _ = one(comms, jobs, n, ncoll, 1, seed, 99, 0.0, "consistent")
                t_cal, _, _ = one(comms, jobs, n, ncoll, 1, seed, 98, 0.0, "consistent")
                mean_gap = t_cal / 1e3 / ncoll
                if wname == "c3" and args.c3_gap == "zero":
                    mean_gap = 0.0
                for rep in range(args.repeats):
                    tc, sc, rc = one(comms, jobs, n, ncoll, iters, seed, rep, mean_gap, "consistent")
                    tr, sr, rr = one(comms, jobs, n, ncoll, iters, seed, rep, mean_gap, "random")
                    ic, ir = ideal_of(rc, dur, iters), ideal_of(rr, dur, iters)
                    row = {"tag": args.tag, "knobs": extra, "workload": wname, "variant": vname, "seed": seed, "repeat": rep, "ranks": n,
                           "ncoll": ncoll, "iterations": iters, "mean_gap_us": mean_gap * 1e6,
                           "ms_consistent": tc, "ms_random": tr, "overhead": tr / tc - 1.0,
                           "ideal_ms_consistent": ic, "ideal_ms_random": ir,
                           "overhead_vs_ideal_consistent": tc / ic - 1.0, "overhead_vs_ideal_random": tr / ir - 1.0,
                           "standalone_ms_total": sum(dur.values()),
                           "preempt_consistent": sc["preemptions"], "preempt_random": sr["preemptions"],
                           "launches_random": sr["launches"], "quits_random": sr["quits"],
                           "iter_ms_random_p90": (sorted(rr["iter_ms"])[int(0.9 * (len(rr["iter_ms"]) - 1))]
                                                  if iters > 1 else None)}
                    rows.append(row)
                    fout.write(json.dumps(row) + "\n")
                    fout.flush()
                    print(json.dumps(row), flush=True)
                del bufs, jobs
                torch.cuda.empty_cache()
            occl.destroy_group(comms)
    fout.close()
    summ = []
    for wname in args.workloads.split(","):
        for vname in args.variants.split(","):
            rs = [r for r in rows if r["workload"] == wname and r["variant"] == vname]
            if not rs:
                continue
            ov = sorted(r["overhead"] for r in rs)
            summ.append({"tag": args.tag, "workload": wname, "variant": vname, "runs": len(rs),
                         "ms_consistent_median": statistics.median(r["ms_consistent"] for r in rs),
                         "ms_random_median": statistics.median(r["ms_random"] for r in rs),
                         "overhead_median": statistics.median(ov), "overhead_min": ov[0], "overhead_max": ov[-1],
                         "overhead_vs_ideal_random_median": statistics.median(r["overhead_vs_ideal_random"] for r in rs),
                         "overhead_vs_ideal_consistent_median": statistics.median(r["overhead_vs_ideal_consistent"]
                                                                                  for r in rs),
                         "preempt_random_median": statistics.median(r["preempt_random"] for r in rs),
                         "preempt_consistent_median": statistics.median(r["preempt_consistent"] for r in rs)})
    with open(args.out + "_summary.json", "w") as f:
        json.dump(summ, f, indent=1)
    for s in summ:
        print("SUMMARY", json.dumps(s), flush=True)


if __name__ == "__main__":
    main()
