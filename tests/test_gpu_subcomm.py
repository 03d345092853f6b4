"""Sub-communicators sharing one daemon per GPU (BASELINE configs[4],
SURVEY.md §8(f) NEXT-2): 8 virtual ranks, tensor-parallel groups {0-3} and
{4-7}, pipeline pairs (i, i+4), plus collectives on the full 8-ring -- all in
flight at once, each rank submitting in its own random order.  Every result is
compared bit-exactly with the oracle run on the sub-communicator's own ring
(child ranks, child size)."""
import random

import pytest
import torch

pytestmark = pytest.mark.gpu

import gpu_util as U  # noqa: E402

CFG = dict(maxColl=64, gridBlocks=4, connSlots=3, slicesPerChunk=2, sliceBytes=32768, minBlockBytes=65536)


@pytest.fixture(scope="module")
def occl_mod():
    if not torch.cuda.is_available():
        pytest.fail("CUDA GPU required for -m gpu tests")
    from paper_2303_06324_b200 import occl
    occl._lib()
    return occl


@pytest.mark.parametrize("policy,ready", [(1, 2), (1, 1), (1, 0), (0, 2)])
def test_overlapping_subcomms_random_orders(occl_mod, policy, ready):
    """Every order policy and readiness-board mode (reading R29: 2 = wait mode,
    1 = spinMin visits, 0 = queue front first; FIFO ignores it)."""
    n = 8
    comms = occl_mod.local_group(n, 0, orderPolicy=policy, readyFirst=ready, spinBase=256, spinStep=32, spinMin=16,
                                 **CFG)
    tp_groups = [[0, 1, 2, 3], [4, 5, 6, 7]]
    pp_groups = [[i, i + 4] for i in range(4)]
    tp = occl_mod.split_group(comms, tp_groups)
    pp = occl_mod.split_group(comms, pp_groups)
    try:
        # (collId, communicator ranks (parent ranks), child comms, kind, dtype, count, root)
        jobs = []
        cid = 0
        for mb in range(3):                                   # interleaved micro-batches
            for gi, g in enumerate(tp_groups):
                jobs.append((cid, g, tp[gi], "allreduce", "bf16", 300_001 + mb, 0)); cid += 1
            for gi, g in enumerate(pp_groups):
                jobs.append((cid, g, pp[gi], "broadcast", "f32", 70_003, mb % 2)); cid += 1
            for gi, g in enumerate(tp_groups):
                jobs.append((cid, g, tp[gi], "allgather", "f32", 20_011, 0)); cid += 1
        jobs.append((cid, list(range(n)), comms, "allreduce", "f32", 1_000_003, 0)); cid += 1
        jobs.append((cid, list(range(n)), comms, "reducescatter", "i32", 50_001, 0)); cid += 1
        bufs = {}
        for j, (c, ranks, cs, kind, dtype, count, root) in enumerate(jobs):
            bufs[c] = U.make_bufs(kind, dtype, len(ranks), count, 500 + c, c)
        # per parent rank: its jobs in a private random order
        rng = random.Random(1234 + policy)
        per_rank = {q: [j for j in jobs if q in j[1]] for q in range(n)}
        for q in range(n):
            rng.shuffle(per_rank[q])
        for q in rng.sample(range(n), n):
            for c, ranks, cs, kind, dtype, count, root in per_rank[q]:
                cr = ranks.index(q)
                s, r = bufs[c][0][cr], bufs[c][1][cr]
                cs[cr].submit(kind, s, r, c, count, dtype, root)
        for c, ranks, cs, kind, dtype, count, root in jobs:
            for child in cs:
                child.wait(c, U.WAIT_S)
        for c, ranks, cs, kind, dtype, count, root in jobs:
            U.check_full(kind, dtype, len(ranks), count, 500 + c, c, bufs[c][1], root)
        st = comms[0].stats()
        assert st["cqeWritten"] >= sum(1 for j in jobs if 0 in j[1])
    finally:
        for group in list(tp.values()) + list(pp.values()):
            for child in group:
                child.destroy()
        occl_mod.destroy_group(comms)


def test_split_errors_and_lifetime(occl_mod):
    comms = occl_mod.local_group(4, 0, **CFG)
    try:
        with pytest.raises(occl_mod.OcclError) as e:
            comms[0].split([1, 2])                            # caller must be a member
        assert e.value.code == occl_mod.occlInvalidArgument
        with pytest.raises(occl_mod.OcclError):
            comms[0].split([0, 0])                            # duplicate member
        kids = [comms[q].split([0, 2]) for q in (0, 2)]
        with pytest.raises(occl_mod.OcclError) as e:
            occl_mod.occlCommDestroy(comms[0].h)              # children first
        assert e.value.code == occl_mod.occlInvalidUsage
        x = [torch.full((1000,), float(q + 1), device=0) for q in range(2)]
        torch.cuda.synchronize()
        for k, t in zip(kids, x):
            k.all_reduce(t, t, 5)
        for k in kids:
            k.wait(5, U.WAIT_S)
        assert torch.all(x[0] == 3.0) and torch.all(x[1] == 3.0)
        for k in kids:
            k.destroy()
    finally:
        occl_mod.destroy_group(comms)


def test_collid_bound_to_first_ring_and_slot_reuse(occl_mod):
    """a collId's connector counters belong to the ring of its
    first submission, so submitting it on another rank set is refused
    (occlInvalidUsage) instead of pairing counters of different edges; a
    destroyed child retires its ids.  Ring slots of destroyed children are
    reused: 40 split / destroy cycles (> 31 slots) all work."""
    comms = occl_mod.local_group(4, 0, **CFG)
    try:
        x = [torch.full((4096,), float(q + 1), device=0) for q in range(4)]
        torch.cuda.synchronize()
        kids = [comms[q].split([0, 1]) for q in (0, 1)]
        for k, t in zip(kids, x):
            k.all_reduce(t, t, 6)
        for k in kids:
            k.wait(6, U.WAIT_S)
        assert torch.all(x[0] == 3.0)
        with pytest.raises(occl_mod.OcclError) as e:
            comms[0].all_reduce(x[2], x[2], 6)               # id 6 is bound to the {0, 1} ring
        assert e.value.code == occl_mod.occlInvalidUsage
        for k in kids:
            k.destroy()
        with pytest.raises(occl_mod.OcclError) as e:
            comms[0].all_reduce(x[2], x[2], 6)               # retired with its ring
        assert e.value.code == occl_mod.occlInvalidUsage
        for cycle in range(40):
            pair = [cycle % 4, (cycle + 1) % 4]
            ks = [comms[q].split(pair) for q in pair]
            y = [torch.full((1000,), float(cycle + i), device=0) for i in range(2)]
            torch.cuda.synchronize()
            for k, t in zip(ks, y):
                k.all_reduce(t, t, 8 + cycle)                 # fresh id per ring
            for k in ks:
                k.wait(8 + cycle, U.WAIT_S)
            assert torch.all(y[0] == float(2 * cycle + 1))
            for k in ks:
                k.destroy()
    finally:
        occl_mod.destroy_group(comms)
