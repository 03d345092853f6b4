#!/usr/bin/env python
"""Per-block timeline of one collective (8 virtual ranks, live daemon, device
trace): for each rank and each of the collective's blocks, fetch / switch-in /
done / CQE of the last repetition, relative to the earliest fetch.  Used to find
which block holds back a collective's completion."""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2303_06324_b200 import harness, occl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kind", default="broadcast")
    ap.add_argument("--bytes", type=int, default=262144)
    ap.add_argument("--reps", type=int, default=6)
    ap.add_argument("--grid", type=int, default=18)
    ap.add_argument("--out", default="gpurun_out/trace_blocks.json")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    n = 8
    comms = harness.ring(n, 0, gridBlocks=a.grid, maxColl=16, traceCap=1 << 14, quitIdleNs=10_000_000_000)
    cid = 1
    count = a.bytes // 4 // (n if a.kind in ("allgather", "reducescatter") else 1)
    bufs = harness.buffers(a.kind, "f32", n, count, comms)
    try:
        for rep in range(a.reps):
            for r, c in enumerate(comms):
                c.submit(a.kind, bufs[r][0], bufs[r][1], cid, count, "f32")
            for c in comms:
                c.wait(cid, 60)
        out = {}
        t0 = None
        for r in range(n):
            for b in range(a.grid):
                tr = comms[r].trace(b)
                fe = [i for i, (t, e, c, x) in enumerate(tr) if e == "fetch" and c == cid]
                if not fe:
                    continue
                ev = {}
                for t, e, c, x in tr[fe[-1]:]:
                    if e in ("fetch", "switch_in", "done", "cqe", "preempt") and (c == cid or e == "fetch"):
                        ev.setdefault(e, []).append(t)
                out[f"r{r}b{b}"] = ev
                t0 = min(t0, ev["fetch"][0]) if t0 is not None else ev["fetch"][0]
        rel = {k: {e: [round((t - t0) / 1e3, 2) for t in ts] for e, ts in v.items()} for k, v in out.items()}
        res = {"kind": a.kind, "bytes": a.bytes, "blocks": rel}
        print(json.dumps(res))
        with open(a.out, "w") as f:
            json.dump(res, f)
    finally:
        occl.destroy_group(comms)


if __name__ == "__main__":
    main()
