"""Asynchronous arrival into a live daemon (PAPER.md:448
"simultaneously arriving collective requests", :816-818 the DP iterations).

Per-rank submitter threads feed the event-driven daemon (autoLaunch = 1,
voluntary quit on) after a barrier; every rank walks its OWN random order with
Exp-distributed gaps between submissions (inputs.workloads.arrival_delays), so
task queues differ across ranks while collectives are running -- the case the
pre-enqueued single-launch runs of round 1 could not show.  Every output is
checked against the oracle (O1); ids are resubmitted every DP iteration right
after local completion."""
import random

import numpy as np
import pytest
import torch

from inputs import workloads
from paper_2303_06324_b200 import harness

import gpu_util as U  # noqa: E402

pytestmark = pytest.mark.gpu

CFG = dict(gridBlocks=8, maxColl=128, sliceBytes=64 << 10, connSlots=4, slicesPerChunk=2, quitIdleNs=500_000)


@pytest.fixture(scope="module")
def occl_mod():
    if not torch.cuda.is_available():
        pytest.fail("CUDA GPU required for -m gpu tests")
    from paper_2303_06324_b200 import occl
    occl._lib()
    return occl


def _jobs(colls, n, seed):
    bufs = {c.coll_id: U.make_bufs(c.kind, c.dtype, n, c.count, seed, c.coll_id) for c in colls}
    jobs = [(c.coll_id, c.kind, c.dtype, c.count, c.root,
             [(bufs[c.coll_id][0][r], bufs[c.coll_id][1][r]) for r in range(n)]) for c in colls]
    return jobs, bufs


@pytest.mark.parametrize("policy,stick", [(1, 1), (0, 1), (0, 0)])
def test_live_c3_scaled_random_orders_and_jitter(occl_mod, policy, stick):
    """C3 shape scaled 1/64 (16 KiB .. 1 MiB), 32 mixed collectives, 8 ranks."""
    n = 8
    comms = occl_mod.local_group(n, 0, orderPolicy=policy, stickiness=stick, **CFG)
    try:
        for seed in range(2):
            colls, orders = workloads.c3(n, 32, seed, scale=64)
            jobs, bufs = _jobs(colls, n, 700 + seed)
            delays = workloads.arrival_delays(n, len(colls), 50e-6, seed)
            before = sum(c.stats()["preemptions"] for c in comms)
            r = harness.live_run(comms, jobs, orders, delays, timeout_s=120)
            assert r["makespan_ms"] > 0
            for c in colls:
                U.check_full(c.kind, c.dtype, n, c.count, 700 + seed, c.coll_id, bufs[c.coll_id][1], c.root)
            _ = sum(c.stats()["preemptions"] for c in comms) - before
    finally:
        occl_mod.destroy_group(comms)


def test_live_c4_resnet_buckets_iterations(occl_mod):
    """C4: ResNet-50 25 MiB buckets, 20 DP iterations; each iteration every rank
    submits the buckets in its own random order with Exp gaps and waits for
    them (ids resubmitted every iteration)."""
    n = 8
    comms = occl_mod.local_group(n, 0, **CFG)
    try:
        colls, _ = workloads.c4("resnet50", n, 0)
        jobs, bufs = _jobs(colls, n, 33)
        r = harness.live_run(comms, jobs, None, None, iterations=20,
                             orders_fn=lambda it: workloads.iteration_orders(n, len(colls), 1, it),
                             delays_fn=lambda it: workloads.arrival_delays(n, len(colls), 100e-6, it))
        assert len(r["iter_ms"]) == 20
        for c in colls:
            U.check_full(c.kind, c.dtype, n, c.count, 33, c.coll_id, bufs[c.coll_id][1], c.root)
        st = comms[0].stats()
        assert st["cqeWritten"] >= 20 * len(colls)
    finally:
        occl_mod.destroy_group(comms)


def test_live_campaign_with_preemptions(occl_mod):
    """The deadlock campaign with live jittered arrival (priority policy): 8 ARs
    of 256 B .. 1 MiB per trial, independent orders and gaps per rank; every
    trial completes, sampled trials are checked; preemptions do occur."""
    n = 8
    comms = occl_mod.local_group(n, 0, **dict(CFG, maxColl=16, spinBase=256, spinStep=32, spinMin=16))
    try:
        pre0 = sum(c.stats()["preemptions"] for c in comms)
        for trial in range(60):
            colls, orders = workloads.deadlock_trial(n, 8, seed=10_000 + trial)
            jobs, bufs = _jobs(colls, n, trial)
            delays = workloads.arrival_delays(n, 8, 30e-6, trial)
            harness.live_run(comms, jobs, orders, delays, timeout_s=60)
            if trial % 10 == 0:
                for c in colls:
                    U.check_full("allreduce", "f32", n, c.count, trial, c.coll_id, bufs[c.coll_id][1])
        assert sum(c.stats()["preemptions"] for c in comms) - pre0 > 0
    finally:
        occl_mod.destroy_group(comms)
