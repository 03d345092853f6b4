"""Pins for O2 (oracle/dfce.py): the paper's scheduling semantics (-m "not gpu").

* deadlock freedom by brute force over ALL per-rank submission orders,
* the NCCL-like baseline fails on exactly the non-identical order sets (invariant I6),
* exact resume: per-(lane, step) transfer counts equal the plan,
* exactly-once completion,
* Fig. 1(b)/(c) scenarios and quit/restart,
* SPEC worked examples for actions and thresholds (tests/golden/spec_examples.json).
"""
import itertools
import json
import os

import numpy as np
import pytest

from inputs import workloads
from oracle import dfce, ring

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _bits(a):
    a = np.asarray(a)
    return a.view({8: np.uint64, 4: np.uint32, 2: np.uint16}[a.dtype.itemsize])


def _check_results(sim, bufs, metas, n, iterations=1):
    for it in range(iterations):
        for m in metas:
            xs = [bufs[(r, m.coll_id, it)][0] for r in range(n)]
            if m.inplace and m.kind in ("allreduce", "broadcast"):
                return  # inputs were overwritten in place; checked elsewhere
            exp = ring.result_full(m.kind, m.dtype, xs, root=m.root)
            for r in range(n):
                got = sim.results[(r, m.coll_id, it)]
                assert np.array_equal(_bits(got), _bits(exp[r])), (m, r, it)


def _check_accounting(sim, metas, n, iterations=1):
    """Exactly-once CQE/callback per submission (I5) and exact transfer counts (I2)."""
    for r in range(n):
        assert len(sim.ranks[r].cq) == sim.ranks[r].submitted
        for m in metas:
            assert sim.callbacks[(r, m.coll_id)] == iterations
    for it in range(iterations):
        for m in metas:
            plan = dfce.plan_transfers(m, n, sim.cfg)
            for (r, b, j), cnt in plan.items():
                assert sim.transfers[(r, m.coll_id, it, b, j)] == cnt, (m, r, b, j)


# ------------------------------------------------------------------ SPEC examples
@pytest.mark.parametrize("ex", GOLDEN["actions"], ids=lambda e: e["prim"])
def test_action_sets(ex):
    inc = None if ex["incoming"] is None else np.array(ex["incoming"], dtype=np.int32)
    loc = None if ex["local"] is None else np.array(ex["local"], dtype=np.int32)
    to_recv, to_send = dfce.apply_action_set(ex["prim"], inc, loc, "i32")
    assert (None if to_recv is None else to_recv.tolist()) == ex["to_recv"], ex["cite"]
    assert (None if to_send is None else to_send.tolist()) == ex["to_send"], ex["cite"]


def test_threshold_formulas():
    g = GOLDEN["thresholds"]
    cfg = dfce.SimConfig(spin_base=g["base"], spin_step=g["step"], spin_min=g["min"],
                         spin_boost=g["boost"], spin_cap=g["cap"])
    for pos, T in g["initial"]:
        assert dfce.initial_threshold(pos, cfg) == T, g["cite"]
    for T0, T1 in g["boost_cases"]:
        assert dfce.boosted_threshold(T0, cfg) == T1, g["cite"]
    # monotone non-increasing in position
    Ts = [dfce.initial_threshold(p, cfg) for p in range(100)]
    assert all(a >= b for a, b in zip(Ts, Ts[1:]))
    off = dfce.SimConfig(stickiness=False)
    assert dfce.initial_threshold(50, off) == off.spin_base
    assert dfce.boosted_threshold(100, off) == 100


def test_connector_capacity_guard():
    with pytest.raises(ValueError):
        dfce.Simulator(2, dfce.SimConfig(K=4, slices_per_chunk=4))


# ------------------------------------------------------------------ geometry coverage
@pytest.mark.parametrize("kind", ring.KINDS)
def test_geometry_covers_every_element_once(kind):
    for n in (1, 2, 3, 5):
        for count in (1, 5, 64, 333, 1000):
            for lanes in (1, 2, 3):
                cfg = dfce.SimConfig(lanes=lanes, K=3, slice_elems=8, slices_per_chunk=2)
                m = dfce.CollMeta(0, kind, "f32", count, nblocks=lanes)
                for r in range(n):
                    segs, part, nloops = dfce.lane_geometry(m, n, r, cfg)
                    cover = {}
                    for q, (sb, rb, ln) in enumerate(segs):
                        for b in range(lanes):
                            st = dfce._Static(m, r, n, None, segs, part, b, nloops, None, None, 0)
                            for loop in range(nloops):
                                for s in range(cfg.slices_per_chunk):
                                    lo, l2 = dfce.slice_range(st, q, loop, s, cfg)
                                    for e in range(lo, lo + l2):
                                        cover[(q, e)] = cover.get((q, e), 0) + 1
                        for e in range(ln):
                            assert cover.get((q, e)) == 1, (kind, n, count, lanes, q, e)
                    assert sum(cover.values()) == sum(s[2] for s in segs)


# ------------------------------------------------------------------ C1
def _c1_metas():
    colls, orders = workloads.c1()
    return [dfce.CollMeta(c.coll_id, c.kind, c.dtype, c.count) for c in colls], orders


@pytest.mark.parametrize("T", [1, 3, 64, 4096])
def test_c1_opposite_orders_complete(T):
    """C1: 2 ranks, 2 fp32 ARs of 1024 elements in opposite orders complete with exact
    sums and at least one preemption (PAPER.md:736-739 at desk scale)."""
    metas, orders = _c1_metas()
    cfg = dfce.SimConfig(spin_base=T, spin_step=max(1, T // 16), spin_min=1, spin_cap=4 * T, seed=T)
    sim, bufs = dfce.run_orders(metas, orders, cfg, seed=7)
    _check_results(sim, bufs, metas, 2)
    _check_accounting(sim, metas, 2)
    assert sim.total_preemptions() >= 1


def test_c1_rank_indexed_exact_sums():
    metas, orders = _c1_metas()
    sim = dfce.Simulator(2, dfce.SimConfig(spin_base=2, spin_min=1, spin_cap=8, seed=1))
    progs = []
    outs = {}
    for r in range(2):
        p = []
        for cid in orders[r]:
            x = (r * 1024 + np.arange(1024)).astype(np.float32)
            o = np.zeros(1024, np.float32)
            outs[(r, cid)] = o
            p.append(("submit", metas[cid], x, o))
        p += [("wait", 0), ("wait", 1)]
        progs.append(p)
    for r in range(2):
        sim.set_program(r, progs[r])
    sim.run()
    exp = (1024 + 2 * np.arange(1024)).astype(np.float32)
    for k, o in outs.items():
        assert np.array_equal(o, exp)


def test_c1_baseline_deadlocks():
    metas, orders = _c1_metas()
    with pytest.raises(dfce.Deadlock):
        dfce.run_orders(metas, orders, dfce.SimConfig(baseline=True, seed=0), seed=7)


# ------------------------------------------------------------------ brute force orders
def _all_order_sets(n, k):
    perms = list(itertools.permutations(range(k)))
    return list(itertools.product(perms, repeat=n))


def _small_metas(k, dtype="f32"):
    sizes = [40, 96, 13]
    return [dfce.CollMeta(i, "allreduce", dtype, sizes[i % len(sizes)]) for i in range(k)]


_BF_CFG = dict(K=3, slice_elems=8, slices_per_chunk=2, quit_idle=64)


@pytest.mark.parametrize("n,k", [(2, 2), (2, 3), (3, 2), (3, 3)])
def test_bruteforce_all_orders_complete(n, k):
    """Deadlock freedom (I1): every one of the (k!)^n per-rank submission order sets
    completes, outputs bit-exact, exactly once, exact transfer counts."""
    metas = _small_metas(k)
    sets = _all_order_sets(n, k)
    variants = [(T, st) for T in (1, 3, 64) for st in (False, True)]
    for si, orders in enumerate(sets):
        T, st = variants[si % len(variants)]
        cfg = dfce.SimConfig(spin_base=T, spin_step=max(1, T // 8), spin_min=1, spin_cap=4 * T,
                             stickiness=st, seed=si, **_BF_CFG)
        sim, bufs = dfce.run_orders(metas, [list(o) for o in orders], cfg, seed=si)
        _check_results(sim, bufs, metas, n)
        _check_accounting(sim, metas, n)


@pytest.mark.parametrize("mode,scan", [(1, 64), (2, 64), (2, 1)])
@pytest.mark.parametrize("n,k", [(2, 2), (2, 3), (3, 2), (3, 3)])
def test_bruteforce_all_orders_ready_first(n, k, mode, scan):
    """The readiness-board rule (R29: run the highest-priority entry every
    member admitted; a non-ready or non-front pick waits spin_min and is not
    boosted) keeps deadlock freedom: every (k!)^n order set completes, outputs
    bit-exact, exactly once, with the rule actually steering (some switch-in picks
    an entry behind the queue front)."""
    metas = _small_metas(k)
    sets = _all_order_sets(n, k)
    steered = waited = 0
    for si, orders in enumerate(sets):
        T = (1, 3, 64)[si % 3]
        cfg = dfce.SimConfig(spin_base=T, spin_step=max(1, T // 8), spin_min=1, spin_cap=4 * T,
                             stickiness=bool((si // 3) % 2), order_policy="priority", ready_first=mode,
                             ready_scan=scan, seed=si, **_BF_CFG)
        sim, bufs = dfce.run_orders(metas, [list(o) for o in orders], cfg, seed=si)
        _check_results(sim, bufs, metas, n)
        _check_accounting(sim, metas, n)
        steered += sim.ready_picks_behind_front
        waited += sim.ready_waits
    assert steered > 0 or scan == 1                      # a 1-entry window never picks behind the front
    assert (waited > 0) == (mode == 2)


@pytest.mark.parametrize("mode", [1, 2])
def test_subcommunicators_all_orders_ready_first(mode):
    """R29 on overlapping sub-communicator rings: readiness is per ring (its own
    members' admissions); all 216 per-rank order sets complete exactly."""
    n, metas = 3, _sub_metas()
    sets = _sub_order_sets(metas, n)
    for si, orders in enumerate(sets):
        T = (1, 3, 64)[si % 3]
        cfg = dfce.SimConfig(spin_base=T, spin_step=max(1, T // 8), spin_min=1, spin_cap=4 * T,
                             stickiness=bool(si % 2), order_policy="priority", ready_first=mode,
                             seed=si, **_BF_CFG)
        sim, bufs = dfce.run_orders(metas, orders, cfg, seed=si)
        _check_sub_results(sim, bufs, metas, n)
        for r in range(n):
            assert len(sim.ranks[r].cq) == sim.ranks[r].submitted


@pytest.mark.parametrize("n,k", [(2, 2), (2, 3), (3, 2), (3, 3)])
def test_bruteforce_every_variant_small(n, k):
    """Each (threshold, stickiness, policy) variant on a deterministic sample of sets."""
    metas = _small_metas(k)
    sets = _all_order_sets(n, k)
    for T in (1, 3, 64):
        for st in (False, True):
            for pol in ("fifo", "priority"):
                for si in range(0, len(sets), max(1, len(sets) // 6)):
                    cfg = dfce.SimConfig(spin_base=T, spin_step=max(1, T // 8), spin_min=1,
                                         spin_cap=4 * T, stickiness=st, order_policy=pol,
                                         seed=si + 100, **_BF_CFG)
                    sim, bufs = dfce.run_orders(metas, [list(o) for o in sets[si]], cfg, seed=si)
                    _check_results(sim, bufs, metas, n)
                    _check_accounting(sim, metas, n)


@pytest.mark.parametrize("n,k", [(2, 2), (2, 3), (3, 2)])
def test_baseline_fails_exactly_on_nonidentical_orders(n, k):
    """I6: non-preemptive, in-order, single-slot execution completes iff all ranks use
    the same order -- k! of the (k!)^n sets pass (Fig. 1(a))."""
    metas = _small_metas(k)
    passed = 0
    for orders in _all_order_sets(n, k):
        same = all(o == orders[0] for o in orders)
        cfg = dfce.SimConfig(baseline=True, seed=1, **_BF_CFG)
        try:
            dfce.run_orders(metas, [list(o) for o in orders], cfg, seed=3)
            ok = True
        except dfce.Deadlock:
            ok = False
        assert ok == same, orders
        passed += ok
    import math
    assert passed == math.factorial(k)


# ------------------------------------------------------------------ Fig. 1(b), 1(c), quit/restart
def test_fig1b_resource_depletion():
    """Fig. 1(b): with S=2 resident 'streams' per rank, 4 collectives started in orders
    whose first two are disjoint deadlock the baseline (every stream busy-waits on a
    collective the peer has no stream left for); S=3 forces the resident sets to
    intersect and passes (control); OCCL's single daemon multiplexes all of them.
    (SPEC.md:511 asks for 3 collectives with S=2, but by pigeonhole two ranks' 2-of-3
    resident sets always intersect, so that case cannot deadlock.)"""
    metas = _small_metas(4)
    orders = [[0, 1, 2, 3], [2, 3, 0, 1]]
    with pytest.raises(dfce.Deadlock):
        dfce.run_orders(metas, orders, dfce.SimConfig(baseline=True, baseline_slots=2, **_BF_CFG))
    dfce.run_orders(metas, orders, dfce.SimConfig(baseline=True, baseline_slots=3, **_BF_CFG))
    sim, bufs = dfce.run_orders(metas, orders, dfce.SimConfig(spin_base=8, spin_min=1, spin_cap=32, **_BF_CFG))
    _check_results(sim, bufs, metas, 2)


def test_fig1c_sync_operation():
    """Fig. 1(c): both ranks start A/B in opposite orders and device-synchronise after
    the first; voluntary quit lets the sync return and both complete."""
    metas = _small_metas(2)
    orders = [[0, 1], [1, 0]]
    cfg = dfce.SimConfig(spin_base=8, spin_min=1, spin_cap=32, **_BF_CFG)
    sim, bufs = dfce.run_orders(metas, orders, cfg, sync_after_first=True)
    _check_results(sim, bufs, metas, 2)
    _check_accounting(sim, metas, 2)
    assert sum(sim.quits) >= 2 and min(sim.launches) >= 2
    with pytest.raises(dfce.Deadlock):
        dfce.run_orders(metas, orders, dfce.SimConfig(baseline=True, **_BF_CFG), sync_after_first=True)
    # without voluntary quit the OCCL daemon itself cannot get past the sync
    with pytest.raises(dfce.Deadlock):
        dfce.run_orders(metas, orders, dfce.SimConfig(quit_enabled=False, spin_base=8, spin_min=1,
                                                      spin_cap=32, **_BF_CFG), sync_after_first=True)


def test_quit_restart_with_delayed_peer():
    """A peer that submits long after the others: blocks quit, contexts survive in the
    context buffer, the event-driven restart completes everything exactly once."""
    metas = _small_metas(3)
    n = 3
    sim = dfce.Simulator(n, dfce.SimConfig(spin_base=4, spin_min=1, spin_cap=16, stall_limit=1,
                                            **_BF_CFG))
    bufs = {}
    for m in metas:
        xs, outs = dfce.make_buffers(m, n, 5)
        for r in range(n):
            bufs[(r, m.coll_id, 0)] = (xs[r], outs[r])
    for r in range(n):
        prog = [("delay", 200_000)] if r == 2 else []
        prog += [("submit", m, *bufs[(r, m.coll_id, 0)]) for m in metas]
        prog += [("wait", m.coll_id) for m in metas]
        sim.set_program(r, prog)
    sim.run()
    _check_results(sim, bufs, metas, n)
    _check_accounting(sim, metas, n)
    assert sim.quits[0] >= 1 and sim.launches[0] >= 2


def test_exit_sqe_drains_then_exits():
    metas = _small_metas(2)
    n = 2
    sim = dfce.Simulator(n, dfce.SimConfig(quit_enabled=False, spin_base=4, spin_min=1, spin_cap=16, **_BF_CFG))
    bufs = {}
    for m in metas:
        xs, outs = dfce.make_buffers(m, n, 5)
        for r in range(n):
            bufs[(r, m.coll_id, 0)] = (xs[r], outs[r])
    for r in range(n):
        order = [0, 1] if r == 0 else [1, 0]
        sim.set_program(r, [("submit", metas[c], *bufs[(r, c, 0)]) for c in order] + [("exit",), ("sync",)])
    sim.run()
    _check_results(sim, bufs, metas, n)
    assert all(not R.alive for R in sim.ranks)


# ------------------------------------------------------------------ multi-lane, mixed, resubmission
def test_multilane_mixed_kinds_random_orders():
    """C3 at desk scale: 4 ranks, 3 lanes, 8 mixed collectives (AR/AG/RS/BC, f32/bf16/i32,
    per-collective block counts), independent random orders, 3 iterations reusing ids."""
    rng = np.random.default_rng(0)
    n, k = 4, 8
    kinds = ["allreduce", "allgather", "reducescatter", "broadcast"]
    metas = [dfce.CollMeta(i, kinds[i % 4], ["f32", "bf16", "i32"][i % 3], int(rng.integers(1, 300)),
                           root=i % n, nblocks=1 + i % 3) for i in range(k)]
    orders = [list(rng.permutation(k)) for _ in range(n)]
    cfg = dfce.SimConfig(lanes=3, K=3, slice_elems=16, slices_per_chunk=2, spin_base=16,
                         spin_step=2, spin_min=1, spin_cap=64, seed=4)
    sim, bufs = dfce.run_orders(metas, orders, cfg, seed=9, iterations=3)
    _check_results(sim, bufs, metas, n, iterations=3)
    _check_accounting(sim, metas, n, iterations=3)


def test_misorder_pairwise_reversed_scaled():
    """PAPER.md:736-739 scaled: 4 ranks, 8 ARs, adjacent pairs reversed,
    several iterations; no dedicated stickiness policy (constant threshold)."""
    n, k = 4, 8
    sizes = [64, 128, 256, 512, 1024, 2048, 4096, 16384]      # bytes, 256 B .. 16 KiB
    metas = [dfce.CollMeta(i, "allreduce", "f32", sizes[i] // 4) for i in range(k)]
    orders = workloads.pairwise_reversed_orders(n, k)
    cfg = dfce.SimConfig(stickiness=False, spin_base=32, spin_min=1, spin_cap=128,
                         K=3, slice_elems=64, slices_per_chunk=2, seed=5)
    sim, bufs = dfce.run_orders(metas, orders, cfg, seed=2, iterations=4)
    _check_results(sim, bufs, metas, n, iterations=4)
    _check_accounting(sim, metas, n, iterations=4)
    assert sim.total_preemptions() > 0


def test_context_cache_and_lazy_save_accounting():
    """Lazy save: saves <= preemptions; direct-mapped cache
    (PAPER.md:513): loads < switch-ins when the ways are not contended."""
    metas = _small_metas(3)
    orders = [[0, 1, 2], [2, 1, 0], [1, 2, 0]]
    cfg = dfce.SimConfig(spin_base=2, spin_min=1, spin_cap=8, cache_ways=4, **_BF_CFG)
    sim, _ = dfce.run_orders(metas, orders, cfg, seed=1)
    assert sim.saves <= sim.total_preemptions()
    assert sim.loads >= 1


# ------------------------------------------------------------------ sub-communicators
def _sub_metas():
    """Overlapping rings on 3 ranks: A = {0,1}, B = {1,2}, C = {2,0} (a cycle of
    pairwise groups) and D = all ranks -- every pair of groups overlaps."""
    return [dfce.CollMeta(0, "allreduce", "f32", 40, members=(0, 1)),
            dfce.CollMeta(1, "allreduce", "i32", 33, members=(1, 2)),
            dfce.CollMeta(2, "allgather", "f32", 9, members=(2, 0)),
            dfce.CollMeta(3, "reducescatter", "bf16", 12)]


def _sub_order_sets(metas, n):
    per_rank = [[m.coll_id for m in metas if r in dfce.ring_members(m, n)] for r in range(n)]
    return [list(map(list, combo)) for combo in itertools.product(*[itertools.permutations(p) for p in per_rank])]


def _check_sub_results(sim, bufs, metas, n):
    for m in metas:
        mem = dfce.ring_members(m, n)
        xs = [bufs[(r, m.coll_id, 0)][0] for r in mem]
        exp = ring.result_full(m.kind, m.dtype, xs, root=m.root)   # the sub-ring's own O1 result
        for k, r in enumerate(mem):
            got = sim.results[(r, m.coll_id, 0)]
            assert np.array_equal(_bits(got), _bits(exp[k])), (m.coll_id, r)


def test_subcommunicators_all_orders_complete():
    """Overlapping sub-communicator rings on one daemon per rank: every per-rank
    order set (each rank orders only its own collectives) completes with the
    sub-ring's exact result, exactly once (liveness I1 holds per ring; admission I4
    is per rank)."""
    n, metas = 3, _sub_metas()
    sets = _sub_order_sets(metas, n)
    assert len(sets) == 6 ** 3
    for si, orders in enumerate(sets):
        T = (1, 3, 64)[si % 3]
        cfg = dfce.SimConfig(spin_base=T, spin_step=max(1, T // 8), spin_min=1, spin_cap=4 * T,
                             stickiness=bool(si % 2), order_policy=("fifo", "priority")[(si // 2) % 2],
                             seed=si, **_BF_CFG)
        sim, bufs = dfce.run_orders(metas, orders, cfg, seed=si)
        _check_sub_results(sim, bufs, metas, n)
        for r in range(n):
            assert len(sim.ranks[r].cq) == sim.ranks[r].submitted
        for m in metas:
            plan = dfce.plan_transfers(m, n, sim.cfg)
            for (r, b, j), cnt in plan.items():
                assert sim.transfers[(r, m.coll_id, 0, b, j)] == cnt


def test_subcommunicators_baseline_deadlocks_on_cyclic_orders():
    """Negative control: the NCCL-like baseline deadlocks when the pairwise groups
    are started in a cyclic order (0 waits for 1 on A, 1 for 2 on B, 2 for 0 on C)
    -- the hybrid-parallel hazard sub-communicators bring -- and completes when all
    ranks follow one global order."""
    n = 3
    metas = _sub_metas()[:3]
    cyclic = [[0, 2], [1, 0], [2, 1]]       # rank 0: A then C; rank 1: B then A; rank 2: C then B
    with pytest.raises(dfce.Deadlock):
        dfce.run_orders(metas, cyclic, dfce.SimConfig(baseline=True, seed=1, **_BF_CFG), seed=2)
    consistent = [[0, 2], [0, 1], [1, 2]]   # ids ascending on every rank
    sim, bufs = dfce.run_orders(metas, consistent, dfce.SimConfig(baseline=True, seed=1, **_BF_CFG), seed=2)
    _check_sub_results(sim, bufs, metas, n)
    sim, bufs = dfce.run_orders(metas, cyclic, dfce.SimConfig(seed=1, **_BF_CFG), seed=2)   # OCCL: fine
    _check_sub_results(sim, bufs, metas, n)


@pytest.mark.parametrize("ways", [1, 2, 4])
def test_cache_conflict_eviction_saves_progressed_context(ways):
    """A direct-mapped way shared by two collectives (ids 0 and 4 at 4 ways), the
    priority policy admitting new SQEs between micro-steps of a run: the context
    switched out of the way must be saved lazily, else it
    resumes from stale progress and the ranks' slices disagree.  Found by timing
    O2 on a scaled C3 (scripts/oracle_timing.py)."""
    spec = [("broadcast", "f32", 509, 1), ("reducescatter", "f32", 204, 0), ("broadcast", "f32", 10108, 7),
            ("reducescatter", "bf16", 2085, 0), ("allreduce", "bf16", 1118, 0)]
    metas = [dfce.CollMeta(i, *s) for i, s in enumerate(spec)]
    cfg = dfce.SimConfig(order_policy="priority", cache_ways=ways, seed=1)
    sim, bufs = dfce.run_orders(metas, [[4, 0, 1, 2, 3]] * 8, cfg, seed=3)
    _check_results(sim, bufs, metas, 8)
    _check_accounting(sim, metas, 8)
    assert sim.saves >= 1
