#!/usr/bin/env python
"""C2 (BASELINE.json configs[1]): single-collective size sweep for AR / AG / RS / BC
on an R-rank ring (default 8 virtual ranks on one B200, one fused daemon).

Per point, two timings:
  * pipelined device time: K collectives on distinct ids in one daemon launch,
    CUDA events on the daemon stream, divided by K (nccl-tests style);
  * end-to-end latency: host clock from submit to occlWait, one at a time,
    through the event-driven daemon (median of 20).
Sizes follow nccl-tests: S = per-rank buffer (AR/BC), total output (AG),
total input per rank (RS).  fp32 sum.  Output: JSON lines + a markdown table.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2303_06324_b200 import harness  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ranks", type=int, default=8)
    ap.add_argument("--min-bytes", type=int, default=4096)
    ap.add_argument("--max-bytes", type=int, default=1 << 30)
    ap.add_argument("--factor", type=int, default=4)
    ap.add_argument("--kinds", default="allreduce,allgather,reducescatter,broadcast")
    ap.add_argument("--out", default="gpurun_out/c2_sweep")
    ap.add_argument("--grid-blocks", type=int, default=18)
    ap.add_argument("--conn-slots", type=int, default=5, help="connector slots K (bench configuration: 5)")
    ap.add_argument("--ll-max", type=int, default=64 << 10, help="LL protocol threshold (per-block part bytes)")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    n = args.ranks
    comms = harness.ring(n, 0, gridBlocks=args.grid_blocks, maxColl=128, autoLaunch=0, llMaxBytes=args.ll_max,
                         connSlots=args.conn_slots)
    rows = []
    sizes = []
    s = args.min_bytes
    while s <= args.max_bytes:
        sizes.append(s)
        s *= args.factor
    for kind in args.kinds.split(","):
        for S in sizes:
            isz = 4
            if kind in ("allgather", "reducescatter"):
                count = max(1, S // (n * isz))
            else:
                count = max(1, S // isz)
            bufs = harness.buffers(kind, "f32", n, count, comms)
            K = int(min(64, max(4, (1 << 31) // (S * n))))
            jobs = [(k, kind, "f32", count, 0, bufs) for k in range(K)]
            harness.timed_batch(comms, jobs)                      # warm-up
            ms = min(harness.timed_batch(comms, jobs) for _ in range(2)) / K
            lat = harness.host_latency(comms, (100, kind, "f32", count, 0, bufs), reps=20)
            algbw = S / (ms / 1e3) / 1e9
            row = {"kind": kind, "bytes": S, "count": count, "ranks": n, "ops_per_launch": K,
                   "device_us": ms * 1e3, "algbw_GBps": algbw,
                   "busbw_GBps": algbw * harness.busbw_factor(kind, n), "e2e_latency_us": lat * 1e3}
            rows.append(row)
            print(json.dumps(row), flush=True)
            del bufs
            torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out + ".jsonl", "w") as f:
        for r in rows:
            f.write(json.dumps(r) + "\n")
    with open(args.out + ".md", "w") as f:
        f.write(f"| kind | bytes | device us/op | algbw GB/s | busbw GB/s | e2e latency us |\n|---|---|---|---|---|---|\n")
        for r in rows:
            f.write(f"| {r['kind']} | {r['bytes']} | {r['device_us']:.1f} | {r['algbw_GBps']:.1f} | "
                    f"{r['busbw_GBps']:.1f} | {r['e2e_latency_us']:.1f} |\n")
    harness.occl.destroy_group(comms)


if __name__ == "__main__":
    main()
