#!/usr/bin/env python
"""C3 (BASELINE.json configs[2]): 8 ranks, 64 concurrent mixed collectives
(AR/AG/RS/BC, fp32/bf16, 1-64 MiB log-uniform) submitted in independent random
per-rank orders vs one consistent order, stickiness on vs off.

Each variant pre-enqueues all 64 SQEs on every rank (each rank in its order)
and runs ONE daemon launch; makespan = device time of that launch (CUDA
events on the daemon stream).  Reports preemptions / context loads / saves.
preemption overhead = T(random) / T(consistent) - 1.
Also C4 (configs[3]): DP gradient buckets (ResNet-50 / BERT-large, 25 MiB
buckets, and the 161 per-tensor ResNet-50 ARs) with per-rank random orders.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from inputs import workloads  # noqa: E402
from paper_2303_06324_b200 import harness, occl  # noqa: E402


def run_variant(comms, colls, orders, bufs):
    before = [c.stats() for c in comms]
    jobs = [(c.coll_id, c.kind, c.dtype, c.count, c.root, bufs[c.coll_id]) for c in colls]
    ms = harness.timed_batch(comms, jobs, orders)
    after = [c.stats() for c in comms]
    d = {k: sum(a[k] - b[k] for a, b in zip(after, before)) for k in ("preemptions", "ctxLoads", "ctxSaves",
                                                                      "slices", "quits", "cqeWritten")}
    return ms, d


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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ranks", type=int, default=8)
    ap.add_argument("--seeds", type=int, default=3)
    ap.add_argument("--workloads", default="c3,resnet50-buckets,resnet50-tensors,bert-large-buckets")
    ap.add_argument("--out", default="gpurun_out/c3_c4")
    ap.add_argument("--spin-ns", type=int, default=0, help="0 = library default")
    ap.add_argument("--variants", default="priority:1,fifo:1,fifo:0",
                    help="order_policy:stickiness pairs")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    n = args.ranks
    rows = []
    for wname in args.workloads.split(","):
        for var in args.variants.split(","):
            pol, stick = var.split(":")
            policy, stick = (1 if pol == "priority" else 0), int(stick)
            comms = harness.ring(n, 0, gridBlocks=18, maxColl=256, autoLaunch=0, stickiness=stick,
                                 orderPolicy=policy, **({"spinNs": args.spin_ns} if args.spin_ns else {}))
            for seed in range(args.seeds):
                colls, orders = workload(wname, n, seed)
                bufs = {c.coll_id: harness.buffers(c.kind, c.dtype, n, c.count, comms) for c in colls}
                consistent = [sorted(range(len(colls)))] * n
                # job index == coll_id for these workloads; one untimed run first
                # (first touch of the connector arena and buffers)
                run_variant(comms, colls, consistent, bufs)
                ms_c, st_c = run_variant(comms, colls, consistent, bufs)
                ms_r, st_r = run_variant(comms, colls, orders, bufs)
                nbytes = sum(c.count * harness.ITEM[c.dtype] * (n if c.kind in ("allgather", "reducescatter") else 1)
                             for c in colls)
                row = {"workload": wname, "order_policy": ["fifo", "priority"][policy], "stickiness": stick, "seed": seed, "ranks": n, "ncoll": len(colls),
                       "bytes_per_rank": nbytes, "ms_consistent": ms_c, "ms_random": ms_r,
                       "preemption_overhead": ms_r / ms_c - 1.0,
                       "random": st_r, "consistent": st_c}
                rows.append(row)
                print(json.dumps(row), flush=True)
                del bufs
                torch.cuda.empty_cache()
            occl.destroy_group(comms)
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out + ".jsonl", "w") as f:
        for r in rows:
            f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
