#!/usr/bin/env python
"""The paper's stickiness case study:
the 161 per-tensor ResNet-50 all-reduces on 8 ranks, every rank
in the same reverse-layer order, but ONE rank submits late (a straggler).  The
other ranks' daemons start the collectives, find the straggler absent and
preempt; the stickiness scheme decides how long they wait and
how the ranks re-converge on the same collective.

Per variant (order policy x stickiness): device makespan of the launch,
preemptions, context loads/saves, and -- from the device trace of rank 1,
block 0 -- the context-switch count and the queue length at each switch-in.
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--delay-ms", type=float, default=2.0)
    ap.add_argument("--out", default="gpurun_out/stickiness_case")
    ap.add_argument("--spin-base", type=int, default=4096)
    ap.add_argument("--spin-cap", type=int, default=65536)
    args = ap.parse_args()
    n = 8
    colls, _ = workloads.c4("resnet50", n, 0, per_tensor=True)
    order = list(range(len(colls)))[::-1]               # backward pass: last layer first
    rows = []
    # (policy, stickiness, priority rule): the priority policy with its default
    # priority = collId, and with a user-defined priority = position in the
    # backward-pass submission order (occlSetPriority, globally agreed)
    for policy, stick, prio in ((0, 1, "-"), (0, 0, "-"), (1, 1, "collId"), (1, 1, "submission")):
        comms = harness.ring(n, 0, gridBlocks=16, maxColl=256, autoLaunch=0, orderPolicy=policy,
                             stickiness=stick, traceCap=1 << 15, spinBase=args.spin_base,
                             spinStep=max(1, args.spin_base // 8), spinMin=min(128, args.spin_base),
                             spinCap=args.spin_cap)
        bufs = {c.coll_id: harness.buffers(c.kind, c.dtype, n, c.count, comms) for c in colls}
        if prio == "submission":
            for pos, k in enumerate(order):
                for c in comms:
                    c.set_priority(colls[k].coll_id, pos)
        torch.cuda.synchronize()
        for c in comms:
            c.trace_reset()
        before = [c.stats() for c in comms]
        pb = [c.probes() for c in comms]
        stream = torch.cuda.ExternalStream(comms[0].stream(), device=0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for r in range(1, n):                            # everybody but the straggler
            for k in order:
                c = colls[k]
                s, rv = bufs[c.coll_id][r]
                comms[r].submit(c.kind, s, rv, c.coll_id, c.count, c.dtype, c.root)
        e0.record(stream)
        comms[0].launch()
        e1.record(stream)
        time.sleep(args.delay_ms / 1e3)                  # rank 0 arrives late
        for k in order:
            c = colls[k]
            s, rv = bufs[c.coll_id][0]
            comms[0].submit(c.kind, s, rv, c.coll_id, c.count, c.dtype, c.root)
        for c in comms:
            c.exit()
        for c in comms:
            for cc in colls:
                c.wait(cc.coll_id, 600)
        comms[0].quiesce(600)
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        after = [c.stats() for c in comms]
        d = {k: sum(a[k] - b[k] for a, b in zip(after, before)) for k in ("preemptions", "ctxLoads", "ctxSaves")}
        pa = [c.probes() for c in comms]
        pr = {k: sum(a[k] - b0[k] for a, b0 in zip(pa, pb)) for k in pa[0]}
        d["ctx_load_us"] = pr["cycCtxLoad"] / max(1, pr["nCtxLoad"]) / 1965.0   # SM clock ~1965 MHz
        d["ctx_save_us"] = pr["cycCtxSave"] / max(1, pr["nCtxSave"]) / 1965.0
        tr = comms[1].trace(0)
        sw = [a for t, ev, c, a in tr if ev == "switch_in"]
        pre = sum(1 for t, ev, c, a in tr if ev == "preempt")
        row = {"policy": ["fifo", "priority"][policy], "stickiness": stick, "priority": prio, "delay_ms": args.delay_ms,
               "spin_base": args.spin_base, "spin_cap": args.spin_cap,
               "makespan_ms": ms, "after_straggler_ms": ms - args.delay_ms, **d,
               "rank1_block0": {"switch_ins": len(sw), "preemptions": pre,
                                "max_queue_pos_at_switch_in": max(sw) if sw else 0}}
        rows.append(row)
        print(json.dumps(row), flush=True)
        occl.destroy_group(comms)
        del bufs
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out + ".jsonl", "w") as f:
        for r in rows:
            f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
