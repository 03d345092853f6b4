#!/usr/bin/env python
"""C5 (BASELINE.json configs[4]): hybrid pipeline + tensor
parallelism with overlapping sub-communicators served by ONE daemon per GPU.

8 ranks (virtual ranks on one B200): tensor-parallel groups {0-3}, {4-7}
(stages 0 and 1), pipeline pairs (i, i+4).  GPT-shaped messages: TP all-reduce
of mb x seq x hidden bf16 = 1 x 2048 x 4096 x 2 B = 16 MiB, pipeline transfer of
the same activation as a 2-rank broadcast (stage 0 -> 1 forward, 1 -> 0
backward).  8 micro-batches in a 1F1B schedule; per micro-batch and stage two TP
all-reduces forward and two backward.

Variants (each one daemon launch, device time):
  * schedule order   : every rank submits its collectives in its 1F1B program order;
  * random arrival   : every rank submits in an independent random permutation;
  * consistent ids   : every rank submits in collId order (NCCL-like single order).
Output: JSON lines (makespan ms, preemptions) to --out.
"""
import argparse
import json
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2303_06324_b200 import harness, occl  # noqa: E402


def build(nmb=8, tp_ar_per_pass=2):
    """Jobs: (collId, kind, parent ranks, group key, root, program-order key per stage)."""
    tp = [[0, 1, 2, 3], [4, 5, 6, 7]]
    pp = [[i, i + 4] for i in range(4)]
    jobs = []
    cid = 0
    # 1F1B on 2 stages: stage 0 runs F0 F1 B0 F2 B1 ...; stage 1 runs F0 B0 F1 B1 ...
    for m in range(nmb):
        for direction in ("F", "B"):
            stage_first = 0 if direction == "F" else 1
            for stage in (stage_first, 1 - stage_first):
                for k in range(tp_ar_per_pass):
                    jobs.append(dict(id=cid, kind="allreduce", ranks=tp[stage], group=("tp", stage), root=0,
                                     mb=m, dir=direction, stage=stage, k=k)); cid += 1
                if stage == stage_first:
                    for pi, g in enumerate(pp):       # activation / gradient hand-off between stages
                        jobs.append(dict(id=cid, kind="broadcast", ranks=g, group=("pp", pi),
                                         root=0 if direction == "F" else 1, mb=m, dir=direction, stage=stage,
                                         k=-1)); cid += 1
    return jobs, tp, pp


def program_order(jobs, q):
    """1F1B program order of parent rank q."""
    stage = 0 if q < 4 else 1

    def key(j):
        m, d = j["mb"], j["dir"]
        # 1F1B slot: stage 0: F(m) at 2m, B(m) at 2m+3; stage 1: F(m) at 2m+1, B(m) at 2m+2
        slot = (2 * m + (0 if stage == 0 else 1)) if d == "F" else (2 * m + (3 if stage == 0 else 2))
        return (slot, j["id"])
    return sorted([j for j in jobs if q in j["ranks"]], key=key)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nmb", type=int, default=8)
    ap.add_argument("--mib", type=float, default=16.0)
    ap.add_argument("--seeds", type=int, default=3)
    ap.add_argument("--out", default="gpurun_out/c5_hybrid")
    ap.add_argument("--slice-kib", type=int, default=0, help="0 = library default")
    ap.add_argument("--ll-max", type=int, default=-1, help="-1 = library default")
    ap.add_argument("--policies", default="1,0")
    ap.add_argument("--spin-ns", type=int, default=0, help="0 = library default")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    n = 8
    jobs, tp, pp = build(args.nmb)
    count = int(args.mib * (1 << 20)) // 2
    rows = []
    extra = {}
    if args.slice_kib:
        extra["sliceBytes"] = args.slice_kib << 10
    if args.ll_max >= 0:
        extra["llMaxBytes"] = args.ll_max
    if args.spin_ns:
        extra["spinNs"] = args.spin_ns
    for policy in [int(x) for x in args.policies.split(",")]:
        comms = harness.ring(n, 0, gridBlocks=16, maxColl=256, autoLaunch=0, orderPolicy=policy, **extra)
        subs = {}
        for gi, g in enumerate(tp):
            subs[("tp", gi)] = [comms[q].split(g) for q in g]
        for gi, g in enumerate(pp):
            subs[("pp", gi)] = [comms[q].split(g) for q in g]
        bufs = {}
        for j in jobs:
            g = j["ranks"]
            bufs[j["id"]] = [(torch.empty(count, dtype=torch.bfloat16, device=0),
                              torch.empty(count, dtype=torch.bfloat16, device=0)) for _ in g]
        torch.cuda.synchronize()

        def run(order_of):
            for c in comms:
                c.set_auto_launch(False)
            comms[0].quiesce(600)
            before = [c.stats() for c in comms]
            for q in range(n):
                for j in order_of(q):
                    cr = j["ranks"].index(q)
                    s, r = bufs[j["id"]][cr]
                    subs[j["group"]][cr].submit(j["kind"], s, r, j["id"], count, "bf16", j["root"])
                comms[q].exit()
            st = torch.cuda.ExternalStream(comms[0].stream(), device=0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            comms[0].launch()
            e1.record(st)
            for j in jobs:
                for child in subs[j["group"]]:
                    child.wait(j["id"], 600)
            comms[0].quiesce(600)
            e1.synchronize()
            after = [c.stats() for c in comms]
            return e0.elapsed_time(e1), sum(a["preemptions"] - b["preemptions"] for a, b in zip(after, before))

        run(lambda q: program_order(jobs, q))                      # warm-up
        ms_ids, p_ids = run(lambda q: sorted([j for j in jobs if q in j["ranks"]], key=lambda j: j["id"]))
        ms_prog, p_prog = run(lambda q: program_order(jobs, q))
        for seed in range(args.seeds):
            rng = random.Random(seed)
            orders = {}
            for q in range(n):
                o = program_order(jobs, q)
                rng.shuffle(o)
                orders[q] = o
            ms_rand, p_rand = run(lambda q: orders[q])
            row = {"workload": "c5-hybrid-pp2-tp4", "order_policy": ["fifo", "priority"][policy], "seed": seed,
                   "microbatches": args.nmb, "msg_MiB": args.mib, "ncoll": len(jobs),
                   "ms_consistent_ids": ms_ids, "ms_1f1b_program_order": ms_prog, "ms_random": ms_rand,
                   "preemptions": {"ids": p_ids, "program": p_prog, "random": p_rand},
                   "overhead_random_vs_consistent": ms_rand / ms_ids - 1.0}
            rows.append(row)
            print(json.dumps(row), flush=True)
        for v in subs.values():
            for child in v:
                child.destroy()
        occl.destroy_group(comms)
        del bufs
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out + ".jsonl", "w") as f:
        for r in rows:
            f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
