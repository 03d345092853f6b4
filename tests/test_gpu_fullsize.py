"""GPU parity in the launch configuration bench.py times (SURVEY.md §8(c),
DESIGN.md §4): 192 KiB slices through a 6-stage TMA staging ring, 5 connector slots, publisher lane,
direct mode, L2 discard / evict-first hints -- the data path the headline
number comes from -- plus its variants and guards.

* full oracle comparison (element by element, bit-exact) at sizes the oracle
  materialises in seconds yet that span many slices, loops and a ragged tail;
* sampled comparison at BASELINE's full size (8 ranks x 256 MiB fp32 AR) in the
  exact bench configuration, including every segment / lane / slice boundary;
* direct mode off (connector-only path), two daemon blocks per SM, misaligned
  per-rank buffers (direct sends into a peer buffer of different alignment);
* the device event trace is consistent with the slice counters;
* the occupancy guard refuses a persistent launch that cannot be co-resident
  (a hang would otherwise follow) and surfaces it as occlCudaError."""
import numpy as np
import pytest
import torch

from oracle import ring

pytestmark = pytest.mark.gpu

import gpu_util as U  # noqa: E402

BENCH = dict(gridBlocks=18, sliceBytes=192 << 10, connSlots=5, slicesPerChunk=2, blockThreads=608, pipeDepth=4,
             stagingTiles=6, maxColl=16)


@pytest.fixture(scope="module")
def occl_mod():
    if not torch.cuda.is_available():
        pytest.fail("CUDA GPU required for -m gpu tests")
    from paper_2303_06324_b200 import occl
    occl._lib()
    return occl


def _ring(occl_mod, n, **kw):
    cfg = dict(BENCH)
    cfg.update(kw)
    return occl_mod.local_group(n, 0, **cfg)


@pytest.mark.parametrize("direct,bulk,hints", [(1, 0, 1), (0, 0, 1), (1, 1, 1), (1, 0, 2), (0, 0, 2)])
def test_bench_config_all_kinds_full_check(occl_mod, direct, bulk, hints):
    """direct mode on / off; bulk-store mode (staged tiles leave through
    cp.async.bulk stores issued by the publisher lane); evict-last connector
    stores (l2Hints=2)."""
    n = 8
    comms = _ring(occl_mod, n, directMode=direct, bulkStores=bulk, l2Hints=hints)
    try:
        for ci, (kind, dtype, count) in enumerate([("allreduce", "f32", 3_000_017), ("allreduce", "bf16", 2_500_003),
                                                   ("allreduce", "i32", 1_048_576), ("allgather", "f32", 400_009),
                                                   ("reducescatter", "bf16", 300_007), ("broadcast", "f32", 2_000_001)]):
            root = ci % n
            sends, recvs = U.make_bufs(kind, dtype, n, count, 40 + ci, ci)
            U.run_collective(comms, kind, sends, recvs, ci, count, dtype, root)
            U.check_full(kind, dtype, n, count, 40 + ci, ci, recvs, root)
            del sends, recvs
    finally:
        occl_mod.destroy_group(comms)


def test_bench_config_full_size_sampled(occl_mod):
    """BASELINE configs[1] headline point: 8 ranks x 256 MiB fp32 all-reduce, the
    bench's exact configuration; sampled outputs + every structural boundary."""
    n, count = 8, (256 << 20) // 4
    comms = _ring(occl_mod, n)
    try:
        sends, recvs = U.make_bufs("allreduce", "f32", n, count, 1, 0)
        U.run_collective(comms, "allreduce", sends, recvs, 0, count, "f32", order=[3, 1, 7, 0, 5, 2, 6, 4])
        seg = -(-count // n)
        seg = -(-seg // 4) * 4                               # owner map: L rounded to 16 B
        part = -(-seg // 18)
        part = -(-part // 4) * 4
        E = BENCH["sliceBytes"] // 4
        bnd = set()
        for q in range(n):
            for lane in range(18):
                base = q * seg + lane * part
                for k in range(0, part, E):
                    bnd.update([base + k - 1, base + k, base + k + 1])
        U.check_sampled("allreduce", "f32", n, count, 1, 0, recvs, nsamples=20000, boundaries=sorted(bnd))
    finally:
        occl_mod.destroy_group(comms)


def test_full_size_bf16_and_ragged_kinds_sampled(occl_mod):
    n = 8
    comms = _ring(occl_mod, n)
    try:
        for ci, (kind, dtype, count) in enumerate([("allreduce", "bf16", (64 << 20) + 13),
                                                   ("allgather", "f32", (8 << 20) + 5),
                                                   ("reducescatter", "f32", (8 << 20) + 3),
                                                   ("broadcast", "bf16", (32 << 20) + 1)]):
            sends, recvs = U.make_bufs(kind, dtype, n, count, 90 + ci, ci)
            U.run_collective(comms, kind, sends, recvs, ci, count, dtype, root=5)
            U.check_sampled(kind, dtype, n, count, 90 + ci, ci, recvs, root=5, nsamples=8000)
            del sends, recvs
            torch.cuda.empty_cache()
    finally:
        occl_mod.destroy_group(comms)


def test_two_blocks_per_sm_variant(occl_mod):
    n = 8
    comms = _ring(occl_mod, n, gridBlocks=36, blocksPerSM=2, blockThreads=352, stagingTiles=3,
                  sliceBytes=64 << 10)
    try:
        for ci, kind in enumerate(ring.KINDS):
            count = 1_000_003
            sends, recvs = U.make_bufs(kind, "f32", n, count, 7 + ci, ci)
            U.run_collective(comms, kind, sends, recvs, ci, count, "f32", root=3)
            U.check_full(kind, "f32", n, count, 7 + ci, ci, recvs, root=3)
    finally:
        occl_mod.destroy_group(comms)


@pytest.mark.parametrize("kind", ring.KINDS)
def test_misaligned_buffers_direct_mode(occl_mod, kind):
    """Per-rank element offsets: direct sends target a peer recv buffer whose
    16-B alignment differs from ours (register / scalar paths must take over)."""
    n, count, dtype = 4, 200_003, "f32"
    comms = _ring(occl_mod, n)
    try:
        inl = count * n if kind == "reducescatter" else count
        outl = count * n if kind == "allgather" else count
        sends, recvs = [], []
        for r in range(n):
            so, ro = (r * 3) % 4, (r * 5 + 1) % 4               # element offsets 0..3
            sb = torch.empty(inl + 4, dtype=torch.float32, device=0)
            rb = torch.full((outl + 4,), -1.0, dtype=torch.float32, device=0)
            s = sb[so:so + inl]
            occl_mod.test_fill(s, dtype, 555, 2, r)
            sends.append(s)
            recvs.append(rb[ro:ro + outl])
        torch.cuda.synchronize()
        U.run_collective(comms, kind, sends, recvs, 2, count, dtype, root=2)
        U.check_full(kind, dtype, n, count, 555, 2, recvs, root=2)
    finally:
        occl_mod.destroy_group(comms)


def test_trace_consistent_with_slice_counters(occl_mod):
    n = 4
    comms = _ring(occl_mod, n, gridBlocks=4, traceCap=1 << 14)
    try:
        count = 2_000_000
        sends, recvs = U.make_bufs("allreduce", "f32", n, count, 3, 1)
        for c in comms:
            c.trace_reset()
        before = [c.coll_stats(1)["slices"] for c in comms]
        U.run_collective(comms, "allreduce", sends, recvs, 1, count, "f32")
        U.check_full("allreduce", "f32", n, count, 3, 1, recvs)
        comms[0].quiesce(60)
        for r, c in enumerate(comms):
            slices = c.coll_stats(1)["slices"] - before[r]
            issued = sum(1 for b in range(4) for ev in c.trace(b) if ev[1] == "issue" and ev[2] == 1)
            assert issued == slices, (r, issued, slices)
            evs = [e[1] for e in c.trace(0)]
            assert "switch_in" in evs and "done" in evs
            ts = [e[0] for e in c.trace(0) if e[1] == "issue"]
            assert ts == sorted(ts)                          # one lane's records are in time order
    finally:
        occl_mod.destroy_group(comms)


def test_occupancy_guard_refuses_non_resident_launch(occl_mod):
    """More daemon blocks than can be co-resident: the launch is refused (a
    persistent ring with blocks that never start would hang)."""
    comms = occl_mod.local_group(1, 0, gridBlocks=400, sliceBytes=128 << 10, maxColl=4)
    try:
        x = torch.ones(1 << 20, device=0)
        torch.cuda.synchronize()
        with pytest.raises(occl_mod.OcclError) as e:
            comms[0].all_reduce(x, x, 0)
            comms[0].wait(0, 10)
        assert e.value.code == occl_mod.occlCudaError
    finally:
        occl_mod.destroy_group(comms)                        # a sticky-errored comm can still be destroyed


def test_memory_footprint_report(occl_mod):
    """occlGetFootprint: the arena, flags, LL lines and contexts follow their
    formulas (the paper's 4 MB per block for 1,000 collectives,
    PAPER.md:581, is reading Q15)."""
    comms = _ring(occl_mod, 2, maxColl=32)
    try:
        f = comms[0].footprint()
        M, G, K, s = 32, BENCH["gridBlocks"], BENCH["connSlots"], BENCH["sliceBytes"]
        assert f["connectorData"] == M * G * K * s
        assert f["connectorFlags"] == M * G * 384
        assert f["contexts"] == M * G * 128
        assert f["llLines"] == M * G * K * 2 * comms[0].cfg.llSliceBytes
        assert f["device"] == sum(f[k] for k in ("connectorData", "connectorFlags", "llLines", "contexts", "other"))
        assert abs(f["perBlockPerColl"] - f["device"] / (M * G)) < 1
    finally:
        occl_mod.destroy_group(comms)


def test_connector_only_sys_scope_full_size_sampled(occl_mod):
    """The one-process-per-GPU data path at the bench configuration: every edge
    connector-only with system-scope fences and flags (forceSysScope = 1, as
    across CUDA IPC), 8 x 256 MiB fp32 AR sampled at every structural boundary
    (VERDICT r01 next #4), plus bf16 AR / AG / RS / BC fully checked at ~1-3 M."""
    n, count = 8, (256 << 20) // 4
    comms = _ring(occl_mod, n, forceSysScope=1)
    try:
        sends, recvs = U.make_bufs("allreduce", "f32", n, count, 21, 0)
        U.run_collective(comms, "allreduce", sends, recvs, 0, count, "f32", order=[5, 2, 7, 0, 3, 1, 6, 4])
        seg = -(-(-(-count // n)) // 4) * 4
        part = -(-(-(-seg // 18)) // 4) * 4
        E = BENCH["sliceBytes"] // 4
        bnd = set()
        for q in range(n):
            for lane in range(18):
                base = q * seg + lane * part
                for k in range(0, part, E):
                    bnd.update([base + k - 1, base + k, base + k + 1])
        U.check_sampled("allreduce", "f32", n, count, 21, 0, recvs, nsamples=20000, boundaries=sorted(bnd))
        del sends, recvs
        torch.cuda.empty_cache()
        for ci, (kind, dtype, count) in enumerate([("allreduce", "bf16", 3_000_017), ("allgather", "f32", 400_009),
                                                   ("reducescatter", "f32", 300_007), ("broadcast", "f32", 2_000_001)]):
            sends, recvs = U.make_bufs(kind, dtype, n, count, 30 + ci, 1 + ci)
            U.run_collective(comms, kind, sends, recvs, 1 + ci, count, dtype, root=ci)
            U.check_full(kind, dtype, n, count, 30 + ci, 1 + ci, recvs, root=ci)
            del sends, recvs
    finally:
        occl_mod.destroy_group(comms)


@pytest.mark.parametrize("hints", [3])
def test_bench_config_l2_keep_direct_sends(occl_mod, hints):
    """l2Hints = 3 (direct sends the downstream forwards stay evict-last for one
    hop and are demoted once read): every kind fully checked at the bench config."""
    n = 8
    comms = _ring(occl_mod, n, l2Hints=hints)
    try:
        for ci, (kind, dtype, count) in enumerate([("allreduce", "f32", 3_000_017), ("allgather", "bf16", 400_009),
                                                   ("reducescatter", "f32", 300_007), ("broadcast", "f32", 2_000_001)]):
            sends, recvs = U.make_bufs(kind, dtype, n, count, 80 + ci, ci)
            U.run_collective(comms, kind, sends, recvs, ci, count, dtype, root=ci % n)
            U.check_full(kind, dtype, n, count, 80 + ci, ci, recvs, root=ci % n)
            del sends, recvs
    finally:
        occl_mod.destroy_group(comms)
