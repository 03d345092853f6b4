"""Per-hop latency of the daemon's ring from the device event trace.

Builds the bench's ring (8 virtual ranks, 256 MiB fp32 all-reduce per rank),
runs `--steps` all-reduces with tracing on, and for block `--block` of every
rank pairs each message's publication at rank r (head raised) with the issue of
the slice that consumes it at rank r+1:
  hop      = issue at r+1 - publish at r      (flag propagation + poll + issue)
  service  = publish at r - issue at r         (TMA loads + compute + fence)
  credit   = issue at r (slot reuse) - credit publication at r+1
Writes a JSON summary (medians / p90 in microseconds).
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2303_06324_b200 import harness, occl  # noqa: E402


def events(trace, kind, coll=0):
    """Events of one collective: those between its switch-in and its completion
    on this block (the bench runs the collectives one after the other)."""
    out, live = [], False
    for t, ev, c, a in trace:
        if ev == "switch_in":
            live = c == coll
        elif ev == "done" and c == coll:
            live = False
        if live and ev == kind:
            out.append((t, c, a))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ranks", type=int, default=8)
    ap.add_argument("--size-mib", type=float, default=256)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--block", type=int, default=3)
    ap.add_argument("--grid-blocks", type=int, default=18)
    ap.add_argument("--slice-kib", type=int, default=128)
    ap.add_argument("--stages", type=int, default=6)
    ap.add_argument("--out", default="gpurun_out/trace_ring.json")
    args = ap.parse_args()
    n = args.ranks
    count = int(args.size_mib * (1 << 20)) // 4
    comms = harness.ring(n, 0, gridBlocks=args.grid_blocks, sliceBytes=args.slice_kib << 10, connSlots=4,
                         slicesPerChunk=2, maxColl=16, stagingTiles=args.stages, traceCap=1 << 16, autoLaunch=0)
    bufs = [(torch.empty(count, device=0), torch.empty(count, device=0)) for _ in range(n)]
    for i, (s, _) in enumerate(bufs):
        occl.test_fill(s, "f32", 1, 0, i)
    jobs = [(k, "allreduce", "f32", count, 0, bufs) for k in range(args.steps)]
    harness.timed_batch(comms, jobs)                       # warm-up
    for c in comms:
        c.trace_reset()
    ms = harness.timed_batch(comms, jobs)
    tr = [c.trace(args.block) for c in comms]
    res = {"ms_per_allreduce": ms / args.steps, "block": args.block}
    hops, serv, cred, gaps = [], [], [], []
    for r in range(n):
        nx = (r + 1) % n
        pub = [(t, arg & 0x3fff, (arg >> 16) & 0x3fff) for t, c, arg in events(tr[r], "publish")]
        iss_r = [(t, arg & 0x3fff, (arg >> 14) & 0x3fff, arg >> 28) for t, c, arg in events(tr[r], "issue")]
        iss_n = [(t, arg & 0x3fff, (arg >> 14) & 0x3fff, arg >> 28) for t, c, arg in events(tr[nx], "issue")]
        pub_n = [(t, arg & 0x3fff, (arg >> 16) & 0x3fff) for t, c, arg in events(tr[nx], "publish")]
        ph = np.array([p[0] for p in pub], dtype=np.float64)
        hv = np.array([p[1] for p in pub])
        # messages sent by r: first publish with head >= m+1 (16-bit wrap ignored: short runs)
        for t, ns, nr, act in iss_r:
            if act & 8:
                k = np.searchsorted(np.maximum.accumulate(hv), ns + 1)
                if k < len(ph):
                    serv.append(ph[k] - t)
        hmax = np.maximum.accumulate(hv) if len(hv) else hv
        for t, ns, nr, act in iss_n:
            if act & 1:
                k = np.searchsorted(hmax, nr + 1)
                if k < len(ph):
                    hops.append(t - ph[k])
        # credit: r's send of message m needs credit >= m-K+1 published by r+1
        cv = np.maximum.accumulate(np.array([p[2] for p in pub_n])) if pub_n else np.array([])
        cph = np.array([p[0] for p in pub_n], dtype=np.float64)
        for t, ns, nr, act in iss_r:
            if act & 8 and ns >= 4:
                k = np.searchsorted(cv, ns - 4 + 1)
                if k < len(cph):
                    cred.append(t - cph[k])
        it = np.array([x[0] for x in iss_r], dtype=np.float64)
        if len(it) > 1:
            gaps.extend(np.diff(it).tolist())

    def q(x):
        x = np.asarray(x) / 1e3
        if len(x) == 0:
            return None
        return {"n": int(len(x)), "p10": float(np.percentile(x, 10)), "median": float(np.median(x)),
                "p90": float(np.percentile(x, 90))}
    # fence: sdone -> publish on the same block (same batch, consecutive records)
    fence = []
    for r in range(n):
        last = None
        for t, ev, c, a in tr[r]:
            if ev == "sdone":
                last = t
            elif ev == "publish" and last is not None:
                fence.append(t - last)
                last = None
    # data: issue -> sdone covering that slice (head value >= nsent+1)
    data = []
    for r in range(n):
        sd = [(t, arg & 0x3fff) for t, c, arg in events(tr[r], "sdone")]
        st = np.array([x[0] for x in sd], dtype=np.float64)
        sh = np.maximum.accumulate(np.array([x[1] for x in sd])) if sd else np.array([])
        for t, c, arg in events(tr[r], "issue"):
            ns, act = arg & 0x3fff, arg >> 28
            if act & 8:
                k = np.searchsorted(sh, ns + 1)
                if k < len(st):
                    data.append(st[k] - t)
    res["fence_us(sdone -> publish)"] = None
    res.update({"hop_us(issue@r+1 - publish@r)": q(hops), "service_us(publish@r - issue@r)": q(serv),
                "credit_slack_us(issue@r - credit publish@r+1; negative = waited)": q(cred),
                "issue_gap_us": q(gaps), "fence_us(sdone -> publish)": q(fence),
                "data_us(issue -> sdone)": q(data)})
    print(json.dumps(res, indent=1))
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump({"summary": res, "trace_rank0": tr[0][:4000], "trace_rank1": tr[1][:4000]}, open(args.out, "w"))
    occl.destroy_group(comms)


if __name__ == "__main__":
    main()
