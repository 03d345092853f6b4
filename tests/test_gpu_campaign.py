"""Deadlock campaign (BASELINE north star: 0 deadlocks across 10,000 random
per-rank submission orders at 8 ranks).  Each trial: 8
all-reduces of 256 B .. 1 MiB in independent random per-rank orders on 8
virtual ranks; every trial must complete under a 10 s watchdog and match the
exact int32 sum (order-free closed form, computed independently with torch).

Two policies: the default priority order (globally agreed priority = collId,
reading R10 -- the ranks' queues converge on the same front, so misordered
submissions rarely need a preemption) and the paper's FIFO order with the
stickiness scheme, where random orders force the daemon to
preempt, save and resume collectives -- the mechanism under test."""
import os
import random

import pytest
import torch

from inputs import workloads

pytestmark = pytest.mark.gpu
TRIALS = int(os.environ.get("OCCL_CAMPAIGN_TRIALS", "10000"))


def test_deadlock_campaign_8_ranks():
    _campaign(TRIALS, orderPolicy=1)


def test_deadlock_campaign_8_ranks_fifo_stickiness():
    """The paper's policy: FIFO task queues + stickiness; preemptions must occur."""
    preempt = _campaign(int(os.environ.get("OCCL_CAMPAIGN_FIFO_TRIALS", "1000")), orderPolicy=0, stickiness=1,
                        spinBase=256, spinStep=32, spinMin=16)
    assert preempt > 0


def _campaign(trials, **cfg):
    if not torch.cuda.is_available():
        pytest.fail("CUDA GPU required")
    from paper_2303_06324_b200 import harness, occl
    n, k = 8, 8
    comms = harness.ring(n, 0, gridBlocks=4, maxColl=16, sliceBytes=16384, minBlockBytes=65536, autoLaunch=0, **cfg)
    g = torch.Generator(device="cuda")
    timeouts, preempt = 0, 0
    try:
        for trial in range(trials):
            colls, orders = workloads.deadlock_trial(n, k, seed=trial)
            jobs = []
            for c in colls:
                s = [torch.randint(-2**31, 2**31 - 1, (c.count,), dtype=torch.int32, device=0, generator=g)
                     for _ in range(n)]
                r = [torch.empty(c.count, dtype=torch.int32, device=0) for _ in range(n)]
                jobs.append((c.coll_id, "allreduce", "i32", c.count, 0, list(zip(s, r))))
            # the API contract: send buffers hold their data when the collective is
            # submitted -- the inputs come from torch's stream
            torch.cuda.synchronize()
            try:
                harness.timed_batch(comms, jobs, orders, timeout_s=10.0)
            except occl.OcclError as e:
                if e.code == occl.occlTimeout:
                    timeouts += 1
                    break
                raise
            for cid, kind, dt, count, root, bufs in jobs:
                exp = _wrap_sum([b[0] for b in bufs])
                for b in bufs:
                    assert torch.equal(b[1], exp), (trial, cid)
        preempt = sum(c.stats()["preemptions"] for c in comms)
    finally:
        occl.destroy_group(comms)
    print(f"campaign {cfg}: {trials} trials, {timeouts} timeouts, {preempt} preemptions")
    assert timeouts == 0
    return preempt


def _wrap_sum(ts):
    acc = ts[0].clone()
    for t in ts[1:]:
        acc = acc + t                     # torch int32 addition wraps (two's complement)
    return acc
