"""GPU scheduling semantics through the C-ABI: any per-rank submission order
completes, forced preemption keeps results bit-exact (exact
resume), voluntary quit + event-driven restart,
the device-synchronisation scenario of Fig. 1(c), callbacks
exactly once and the Exiting SQE."""
import os
import random
import subprocess
import sys
import threading
import time

import numpy as np
import pytest
import torch

from inputs import workloads
import gpu_util as U  # noqa: E402

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

BASE = dict(maxColl=32, gridBlocks=4, connSlots=3, slicesPerChunk=2, sliceBytes=8192, minBlockBytes=16384)


@pytest.fixture(scope="module")
def occl_mod():
    if not torch.cuda.is_available():
        pytest.fail("CUDA GPU required for -m gpu tests")
    from paper_2303_06324_b200 import occl
    return occl


def _run_orders(comms, colls, orders, seed, check=True):
    n = len(comms)
    bufs = {}
    for c in colls:
        bufs[c.coll_id] = U.make_bufs(c.kind, c.dtype, n, c.count, seed, c.coll_id)
    # interleave the ranks' submissions round-robin, each rank in its own order
    for k in range(len(colls)):
        for r in range(n):
            c = colls[orders[r][k]]
            s, rv = bufs[c.coll_id]
            comms[r].submit(c.kind, s[r], rv[r], c.coll_id, c.count, c.dtype, c.root)
    for r in range(n):
        for c in colls:
            comms[r].wait(c.coll_id, U.WAIT_S)
    if check:
        for c in colls:
            U.check_full(c.kind, c.dtype, n, c.count, seed, c.coll_id, bufs[c.coll_id][1], c.root)


def test_c1_opposite_orders(occl_mod):
    """C1 on the GPU: 2 ranks, 2 fp32 ARs of 1024 elements, opposite orders."""
    comms = occl_mod.local_group(2, 0, **BASE, spinBase=64, spinStep=4, spinMin=16, spinCap=256)
    try:
        colls, orders = workloads.c1()
        for it in range(20):
            _run_orders(comms, colls, orders, seed=it)
        st = [c.stats() for c in comms]
        assert all(s["cqeWritten"] == 40 for s in st)
    finally:
        occl_mod.destroy_group(comms)


@pytest.mark.parametrize("T,ready", [(1, 2), (8, 2), (4096, 2), (1, 1), (1, 0)])
def test_random_orders_forced_preemption(occl_mod, T, ready):
    """8 ranks, 8 mixed collectives in independent random orders; tiny thresholds
    force constant preemption -- results stay bit-exact (I2 exact resume), under
    every readiness-board mode (R29)."""
    comms = occl_mod.local_group(8, 0, **BASE, readyFirst=ready, spinBase=T, spinStep=1, spinMin=1,
                                 spinCap=max(T, 4 * T))
    try:
        rng = random.Random(T + 7 * ready)
        kinds = ["allreduce", "allgather", "reducescatter", "broadcast"]
        colls = [workloads.Coll(i, kinds[i % 4], ["f32", "bf16", "i32"][i % 3], rng.randint(1, 40_000),
                                root=rng.randrange(8)) for i in range(8)]
        for it in range(3):
            orders = [rng.sample(range(8), 8) for _ in range(8)]
            _run_orders(comms, colls, orders, seed=100 * T + it)
        pre = sum(c.stats()["preemptions"] for c in comms)
        if T == 1 and ready != 2:
            assert pre > 0           # (wait mode runs nothing that cannot complete: it may not preempt)
    finally:
        occl_mod.destroy_group(comms)


@pytest.mark.parametrize("T", [1, 8, 4096])
def test_ll_speculation_random_orders(occl_mod, T):
    """LL speculation (cfg.llSpeculate): recv slices are handed to the data warps
    before their lines arrived; under misordered submissions and tiny thresholds
    the control thread aborts them and redoes them later.  Every collective here
    is LL-sized; results must stay bit-exact and, at T = 1, aborts must happen."""
    comms = occl_mod.local_group(8, 0, **BASE, llSpeculate=1, spinBase=T, spinStep=1, spinMin=1,
                                 spinCap=max(T, 4 * T))
    try:
        rng = random.Random(1000 + T)
        kinds = ["allreduce", "allgather", "reducescatter", "broadcast"]
        colls = [workloads.Coll(i, kinds[i % 4], ["f32", "bf16", "i32"][i % 3], rng.randint(1, 6_000),
                                root=rng.randrange(8)) for i in range(8)]
        for it in range(4):
            orders = [rng.sample(range(8), 8) for _ in range(8)]
            _run_orders(comms, colls, orders, seed=300 * T + it)
        pre = sum(c.stats()["preemptions"] for c in comms)
        if T == 1:
            assert pre > 0
    finally:
        occl_mod.destroy_group(comms)


@pytest.mark.parametrize("T", [1, 8, 4096])
@pytest.mark.parametrize("policy", [0, 1])
def test_ll_runs_random_orders(occl_mod, T, policy):
    """LL runs (cfg.llSpeculate = 2): the compute warps walk a latency-bound
    collective's whole slice schedule and stop when a slice's lines do not come
    within the spin threshold; the control lane takes over the reported cursor
    (preempted runs resume there; partly sent lines are rewritten identically).
    Misordered submissions, tiny thresholds, FIFO and priority policies: results
    bit-exact, and at T = 1 runs are preempted."""
    comms = occl_mod.local_group(8, 0, **BASE, llSpeculate=2, orderPolicy=policy, spinBase=T, spinStep=1,
                                 spinMin=1, spinCap=max(T, 4 * T))
    try:
        rng = random.Random(2000 + T + 7 * policy)
        kinds = ["allreduce", "allgather", "reducescatter", "broadcast"]
        colls = [workloads.Coll(i, kinds[i % 4], ["f32", "bf16", "i32"][i % 3], rng.randint(1, 6_000),
                                root=rng.randrange(8)) for i in range(8)]
        for it in range(4):
            orders = [rng.sample(range(8), 8) for _ in range(8)]
            _run_orders(comms, colls, orders, seed=500 * T + it + 50 * policy)
        pre = sum(c.stats()["preemptions"] for c in comms)
        if T == 1 and policy == 0:
            assert pre > 0
    finally:
        occl_mod.destroy_group(comms)


def test_deadlock_campaign_small(occl_mod):
    """PAPER.md:736-739 at n=8: ARs of 256 B..1 MiB in independent random per-rank
    orders; every trial must complete (0 timeouts) and match the oracle."""
    comms = occl_mod.local_group(8, 0, **dict(BASE, maxColl=16))
    try:
        for trial in range(25):
            colls, orders = workloads.deadlock_trial(8, 8, seed=trial)
            _run_orders(comms, colls, orders, seed=trial, check=(trial % 5 == 0))
    finally:
        occl_mod.destroy_group(comms)


def test_quit_and_event_driven_restart(occl_mod):
    """One rank submits 0.3 s late: the others' daemons quit voluntarily (queue
    stuck, no SQE) and restart; contexts survive in the context buffer."""
    comms = occl_mod.local_group(3, 0, **BASE, quitIdleNs=2_000_000, spinBase=256, spinMin=64, spinCap=1024)
    try:
        n, count = 3, 50_000
        sends, recvs = U.make_bufs("allreduce", "f32", n, count, 4, 0)
        for r in range(2):
            comms[r].submit("allreduce", sends[r], recvs[r], 0, count, "f32")
        time.sleep(0.3)
        comms[2].submit("allreduce", sends[2], recvs[2], 0, count, "f32")
        for c in comms:
            c.wait(0, U.WAIT_S)
        U.check_full("allreduce", "f32", n, count, 4, 0, recvs)
        s0 = comms[0].stats()
        assert s0["quits"] >= 1 and s0["launches"] >= 2
    finally:
        occl_mod.destroy_group(comms)


def test_callbacks_exactly_once(occl_mod):
    comms = occl_mod.local_group(2, 0, **BASE)
    try:
        hits = {0: 0, 1: 0}
        lock = threading.Lock()

        def cb(cid):
            with lock:
                hits[cid] += 1
        for c in comms:
            c.set_callback(0, cb)
            c.set_callback(1, cb)
        for it in range(10):
            sends, recvs = U.make_bufs("allreduce", "f32", 2, 1000, it, 0)
            s2, r2 = U.make_bufs("allgather", "f32", 2, 100, it, 1)
            for r in (1, 0):
                comms[r].submit("allgather", s2[r], r2[r], 1, 100, "f32")
                comms[r].submit("allreduce", sends[r], recvs[r], 0, 1000, "f32")
            for c in comms:
                c.wait(0, U.WAIT_S)
                c.wait(1, U.WAIT_S)
        time.sleep(0.05)
        assert hits == {0: 20, 1: 20}
    finally:
        occl_mod.destroy_group(comms)


def test_exit_sqe_drains_then_restart(occl_mod):
    """Exiting SQE: blocks drain and exit; a later submission restarts the daemon."""
    comms = occl_mod.local_group(2, 0, **BASE, quitEnabled=0)
    try:
        for it in range(3):
            sends, recvs = U.make_bufs("allreduce", "f32", 2, 3000, it, 2)
            for r in range(2):
                comms[r].submit("allreduce", sends[r], recvs[r], 2, 3000, "f32")
                comms[r].exit()
            for c in comms:
                c.wait(2, U.WAIT_S)
                c.quiesce(U.WAIT_S)
            U.check_full("allreduce", "f32", 2, 3000, it, 2, recvs)
        assert all(c.stats()["exits"] >= 3 * 4 for c in comms)
    finally:
        occl_mod.destroy_group(comms)


def test_manual_launch_mode(occl_mod):
    """autoLaunch off: SQEs queue up; occlCommLaunch runs them (bench mode)."""
    comms = occl_mod.local_group(4, 0, **BASE, autoLaunch=0)
    try:
        sends, recvs = U.make_bufs("allreduce", "bf16", 4, 77_777, 8, 5)
        for r in range(4):
            comms[r].submit("allreduce", sends[r], recvs[r], 5, 77_777, "bf16")
            comms[r].exit()
        time.sleep(0.01)
        assert not any(c.test(5) for c in comms)
        for c in comms:
            c.launch()
        for c in comms:
            c.wait(5, U.WAIT_S)
            c.quiesce(U.WAIT_S)
        U.check_full("allreduce", "bf16", 4, 77_777, 8, 5, recvs)
    finally:
        occl_mod.destroy_group(comms)


def test_fig1c_device_sync_scenario():
    """Fig. 1(c): two ranks start A / B in opposite orders and synchronise the device
    after the first; the daemons' voluntary quit lets the sync return.  Run in a
    subprocess under a hard timeout so a regression cannot hang the suite."""
    code = r'''
import sys, torch
sys.path.insert(0, %r)
sys.path.insert(0, %r)
from paper_2303_06324_b200 import occl
import gpu_util as U
comms = occl.local_group(2, 0, maxColl=8, gridBlocks=2, connSlots=3, slicesPerChunk=2, sliceBytes=8192,
                         minBlockBytes=16384, quitIdleNs=1_000_000, spinBase=256, spinMin=64, spinCap=1024)
A = U.make_bufs("allreduce", "f32", 2, 20000, 1, 0)
B = U.make_bufs("allreduce", "f32", 2, 20000, 2, 1)
comms[0].submit("allreduce", A[0][0], A[1][0], 0, 20000, "f32")
comms[1].submit("allreduce", B[0][1], B[1][1], 1, 20000, "f32")
torch.cuda.synchronize()          # device sync between misordered starts
comms[0].submit("allreduce", B[0][0], B[1][0], 1, 20000, "f32")
comms[1].submit("allreduce", A[0][1], A[1][1], 0, 20000, "f32")
for c in comms:
    c.wait(0, 30); c.wait(1, 30)
U.check_full("allreduce", "f32", 2, 20000, 1, 0, A[1])
U.check_full("allreduce", "f32", 2, 20000, 2, 1, B[1])
print("FIG1C_OK", comms[0].stats()["quits"])
occl.destroy_group(comms)
''' % (ROOT, os.path.join(ROOT, 'tests'))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120, cwd=ROOT)
    assert "FIG1C_OK" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("cq_mode", [1, 2])
def test_cq_ring_variants(occl_mod, cq_mode):
    """The paper's ring-buffer CQs as ablations of the id-slot
    CQ: vanilla (entry, fence, in-order tail) and packed 64-bit {stamp, id}.
    Random per-rank orders with forced preemption; results exact, one CQE per
    submission, the CQE-write probe counts them."""
    comms = occl_mod.local_group(4, 0, **BASE, cqMode=cq_mode, spinBase=8, spinStep=1, spinMin=1, spinCap=32)
    try:
        rng = random.Random(cq_mode)
        kinds = ["allreduce", "allgather", "reducescatter", "broadcast"]
        colls = [workloads.Coll(i, kinds[i % 4], "f32", rng.randint(1, 30_000), root=i % 4) for i in range(12)]
        for it in range(4):
            orders = [rng.sample(range(12), 12) for _ in range(4)]
            _run_orders(comms, colls, orders, seed=50 + it)
        for c in comms:
            c.exit()                                          # probes are flushed when the blocks exit
        comms[0].quiesce(U.WAIT_S)
        for c in comms:
            st, pr = c.stats(), c.probes()
            assert st["cqeWritten"] == 48 and pr["nCqe"] == 48 and pr["cycCqe"] > 0
    finally:
        occl_mod.destroy_group(comms)
