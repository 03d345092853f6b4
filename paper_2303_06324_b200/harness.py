"""Benchmark harness helpers on top of the C-ABI binding (no CPU reference code).

* ``ring(...)``        -- R ranks over this process's GPU(s) (virtual ranks fused
                          into one daemon launch) or over torch.distributed.
* ``timed_batch(...)`` -- submit a batch of collectives on every rank (each
                          rank in its own order), push the Exiting SQE, launch
                          the daemon once and time the launch with CUDA events
                          on the daemon's stream (device time).
"""
from __future__ import annotations

import threading
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


def live_run(comms, jobs, orders, delays, iterations=1, timeout_s=300.0, orders_fn=None, delays_fn=None):
    """Asynchronous arrival into a LIVE daemon.

    One submitter thread per local rank.  After a common barrier each thread
    walks its own order, sleeping delays[local][k] before its k-th submission,
    then waits for all of its collectives; with iterations > 1 it repeats
    (ids are resubmitted after local completion, like DP buckets every step).
    The daemon runs event-driven (autoLaunch = 1): it is (re)launched by the
    host supervisor on new SQEs and may quit voluntarily when idle.

    jobs[k] = (coll_id, kind, dtype, count, root, bufs) with bufs[local] = (send, recv).
    orders_fn(it) / delays_fn(it) override orders / delays per iteration.
    Returns {"makespan_ms", "iter_ms": [...], "submit_ms": per-rank submission
    span}; host CLOCK_MONOTONIC (one box, one process)."""
    n = len(comms)
    dev = comms[0].dev
    torch.cuda.current_stream(dev).synchronize()
    for c in comms:
        c.set_auto_launch(True)
    bar = threading.Barrier(n + 1)
    first = [[None] * iterations for _ in range(n)]
    sub_t = [[dict() for _ in range(iterations)] for _ in range(n)]   # [rank][it][job index] -> submit time
    last = [[None] * iterations for _ in range(n)]
    errors = []

    def worker(li):
        c = comms[li]
        try:
            bar.wait()
            for it in range(iterations):
                od = orders_fn(it)[li] if orders_fn else orders[li]
                dl = delays_fn(it)[li] if delays_fn else delays[li]
                t_next = time.perf_counter()
                for pos, k in enumerate(od):
                    t_next += dl[pos]
                    dt = t_next - time.perf_counter()
                    if dt > 0:
                        time.sleep(dt)
                    cid, kind, dtype, count, root, bufs = jobs[k]
                    s, r = bufs[li]
                    if first[li][it] is None:
                        first[li][it] = time.perf_counter()
                    sub_t[li][it][k] = time.perf_counter()
                    c.submit(kind, s, r, cid, count, dtype, root)
                for k in od:
                    c.wait(jobs[k][0], timeout_s)
                last[li][it] = time.perf_counter()
        except Exception as e:  # noqa: BLE001 -- surfaced by the caller
            errors.append((li, e))
            bar.abort()

    ts = [threading.Thread(target=worker, args=(li,), daemon=True) for li in range(n)]
    for t in ts:
        t.start()
    try:
        bar.wait()
    except threading.BrokenBarrierError:
        pass
    for t in ts:
        t.join(timeout_s * max(1, iterations))
    if errors:
        raise errors[0][1]
    if any(t.is_alive() for t in ts):
        raise TimeoutError("live_run: submitter threads did not finish")
    iter_ms = [(max(last[r][it] for r in range(n)) - min(first[r][it] for r in range(n))) * 1e3
               for it in range(iterations)]
    makespan = (max(last[r][-1] for r in range(n)) - min(first[r][0] for r in range(n))) * 1e3
    # per iteration and job: when the LAST rank submitted it (a collective cannot
    # start earlier), relative to the iteration's first submission, in ms
    ready_ms = [{k: (max(sub_t[r][it][k] for r in range(n)) - min(first[r][it] for r in range(n))) * 1e3
                 for k in sub_t[0][it]} for it in range(iterations)]
    return {"makespan_ms": makespan, "iter_ms": iter_ms, "ready_ms": ready_ms}
