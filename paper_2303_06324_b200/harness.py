"""Benchmark harness helpers on top of the C-ABI binding (no CPU reference code).

* ``ring(...)``        -- R ranks over this process's GPU(s) (virtual ranks fused
                          into one daemon launch) or over torch.distributed.
* ``timed_batch(...)`` -- submit a batch of collectives on every rank (each
                          rank in its own order), push the Exiting SQE, launch
                          the daemon once and time the launch with CUDA events
                          on the daemon's stream (device time).
"""
from __future__ import annotations

import time

import torch

from . import occl

TORCH_DT = {"f32": torch.float32, "bf16": torch.bfloat16, "i32": torch.int32, "f16": torch.float16,
            "i64": torch.int64, "f64": torch.float64}
ITEM = {"f32": 4, "bf16": 2, "i32": 4, "f16": 2, "i64": 8, "f64": 8}


def ring(nranks, device=0, dist=None, world=1, prank=0, **cfg):
    """R = nranks ranks; V = nranks // world consecutive ranks in this process."""
    V = nranks // world
    c = occl.occlConfigDefault(**cfg)
    hs = [occl.occlCommCreate(nranks, prank * V + i, device, c) for i in range(V)]
    mine = [occl.occlCommGetHandle(h) for h in hs]
    if dist is not None and world > 1:
        allh = [None] * world
        dist.all_gather_object(allh, mine)
        handles = [h for part in allh for h in part]
    else:
        handles = mine
    for h in hs:
        occl.occlCommConnect(h, handles)
    comms = [occl.Comm(h, nranks, prank * V + i, device, c) for i, h in enumerate(hs)]
    if V > 1:
        occl.occlCommFuse(comms)
    return comms


def buffers(kind, dtype, nranks, count, comms, device=0, fill=None):
    """(send, recv) per local rank following nccl-tests conventions:
    count = AR/BC elements per rank, AG sendcount, RS recvcount."""
    tdt = TORCH_DT[dtype]
    inl = count * nranks if kind == "reducescatter" else count
    outl = count * nranks if kind == "allgather" else count
    out = []
    for c in comms:
        s = torch.empty(inl, dtype=tdt, device=device)
        r = torch.empty(outl, dtype=tdt, device=device)
        if fill is not None:
            fill(s, c.rank)
        out.append((s, r))
    return out


def timed_batch(comms, jobs, orders=None, timeout_s=600.0):
    """jobs: list of (coll_id, kind, dtype, count, root, bufs) with bufs[local] = (send, recv).
    orders[local]: permutation of job indices for that rank (default: same order).
    Returns device milliseconds of the single daemon launch that ran them all."""
    dev = comms[0].dev
    # send buffers must hold their data at submission (occl.h conventions,
    # PAPER.md:525); callers produce them on torch's current stream
    torch.cuda.current_stream(dev).synchronize()
    for c in comms:
        c.set_auto_launch(False)
    comms[0].quiesce(timeout_s)                       # no event-driven daemon still running
    stream = torch.cuda.ExternalStream(comms[0].stream(), device=dev)
    for li, c in enumerate(comms):
        order = orders[li] if orders is not None else range(len(jobs))
        for k in order:
            cid, kind, dtype, count, root, bufs = jobs[k]
            s, r = bufs[li]
            c.submit(kind, s, r, cid, count, dtype, root)
        c.exit()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    comms[0].launch()
    e1.record(stream)
    for c in comms:
        for cid, *_ in jobs:
            c.wait(cid, timeout_s)
    comms[0].quiesce(timeout_s)
    e1.synchronize()
    return e0.elapsed_time(e1)


def host_latency(comms, job, reps=20, timeout_s=60.0):
    """End-to-end latency (host clock, submit -> occlWait return) of one collective
    at a time through the event-driven daemon (autoLaunch on)."""
    cid, kind, dtype, count, root, bufs = job
    for c in comms:
        c.set_auto_launch(True)
    ts = []
    for it in range(reps + 2):
        t0 = time.perf_counter()
        for li, c in enumerate(comms):
            s, r = bufs[li]
            c.submit(kind, s, r, cid, count, dtype, root)
        for c in comms:
            c.wait(cid, timeout_s)
        ts.append(time.perf_counter() - t0)
    for c in comms:
        c.set_auto_launch(False)
    comms[0].quiesce(timeout_s)
    ts = sorted(ts[2:])
    return ts[len(ts) // 2] * 1e3


def busbw_factor(kind, n):
    return {"allreduce": 2 * (n - 1) / n, "allgather": (n - 1) / n, "reducescatter": (n - 1) / n,
            "broadcast": 1.0}[kind]
