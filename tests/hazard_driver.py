#!/usr/bin/env python
"""Subprocess driver of the send-buffer hazard tests (tests/test_gpu_hazards.py).

The occl.h contract lets a caller rewrite its send buffer, or resubmit the same
collective id, as soon as occlWait returned (connectors and
ids are recycled only after the collective is done).  With direct read (the
downstream reads a same-process upstream's send buffer itself)
a rank's local completion must therefore imply that its downstream has
finished reading that buffer.

Scenario (deterministic, n ranks of one fused daemon, FIFO policy):
  * rank 1 -- the downstream of rank 0 -- first submits Y, which nobody else
    has submitted yet, then X; it spins on Y for `spinBase * spinNs` (~20 ms),
    admits X, and spins on Y again before it ever runs X;
  * every other rank submits X at once; rank 0 waits for X;
  * mode scribble : rank 0 overwrites its send buffer right after its wait;
  * mode resubmit : rank 0 also resubmits X at once (new data, new recv
    buffer); the other ranks resubmit X after their first X completed.
  * then every rank submits Y; all X / Y results are checked bit-exactly
    against the oracle (X#1 with the ORIGINAL inputs of rank 0).

A build where rank 0 completes before rank 1 read its buffer fails the check
(scribble) or deadlocks rank 1 (resubmit: rank 0's second admission
overwrites the {sendbuff, subSeq} line rank 1 still needs); the parent test
enforces a hard timeout.  Prints HAZARD_OK on success."""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import gpu_util as U  # noqa: E402
from paper_2303_06324_b200 import occl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kind", default="reducescatter")
    ap.add_argument("--n", type=int, default=2)
    ap.add_argument("--count", type=int, default=200_000)
    ap.add_argument("--mode", default="scribble", choices=["scribble", "resubmit"])
    ap.add_argument("--spin-ns", type=int, default=5000)
    a = ap.parse_args()
    n, kind, count, dt = a.n, a.kind, a.count, "f32"
    X, Y = 1, 0
    comms = occl.local_group(n, 0, maxColl=8, gridBlocks=4, connSlots=5, slicesPerChunk=2, sliceBytes=192 << 10,
                             minBlockBytes=128 << 10, orderPolicy=occl.occlOrderFifo, stickiness=0,
                             spinBase=4096, spinStep=1, spinMin=1, spinCap=4096, spinNs=a.spin_ns, stallLimit=1,
                             quitIdleNs=10_000_000_000)
    try:
        sx, rx = U.make_bufs(kind, dt, n, count, 11, X)
        sy, ry = U.make_bufs("allreduce", dt, n, 4096, 13, Y)
        rx2 = [torch.zeros_like(t) for t in rx]
        torch.cuda.current_stream().synchronize()
        comms[1].submit("allreduce", sy[1], ry[1], Y, 4096, dt)
        comms[1].submit(kind, sx[1], rx[1], X, count, dt)
        for r in range(n):
            if r != 1:
                comms[r].submit(kind, sx[r], rx[r], X, count, dt)
        t0 = time.perf_counter()
        comms[0].wait(X, 30)
        t_done0 = time.perf_counter() - t0
        # rank 0 rewrites its send buffer (allowed once its wait returned)
        occl.test_fill(sx[0], dt, 12, X, 0)
        torch.cuda.current_stream().synchronize()
        if a.mode == "resubmit":
            comms[0].submit(kind, sx[0], rx2[0], X, count, dt)
        for r in range(1, n):
            comms[r].wait(X, 30)
            if a.mode == "resubmit":
                occl.test_fill(sx[r], dt, 12, X, r)
                torch.cuda.current_stream().synchronize()
                comms[r].submit(kind, sx[r], rx2[r], X, count, dt)
        for r in range(n):
            if r != 1:
                comms[r].submit("allreduce", sy[r], ry[r], Y, 4096, dt)
        for c in comms:
            c.wait(Y, 30)
            c.wait(X, 30)
        U.check_full(kind, dt, n, count, 11, X, rx)
        U.check_full("allreduce", dt, n, 4096, 13, Y, ry)
        if a.mode == "resubmit":
            U.check_full(kind, dt, n, count, 12, X, rx2)
        print(f"HAZARD_OK kind={kind} n={n} mode={a.mode} rank0_done_ms={t_done0 * 1e3:.1f}", flush=True)
    finally:
        occl.destroy_group(comms)


if __name__ == "__main__":
    main()
