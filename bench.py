#!/usr/bin/env python
"""Benchmark: all-reduce bus bandwidth of the OCCL daemon path on B200.

Workload (BASELINE.json configs[1], the C2 sweep's headline point): an
all-reduce of S = 256 MiB (--size-mib) of fp32 per rank, sum, out of place.

* N = 1 (default): a ring of R = 8 virtual ranks (--ranks) on the one B200,
  served by ONE fused daemon launch (they share HBM).  Also reported: the
  same ring on the connector-only / system-scope data path a one-process-per-
  GPU ring runs (forceSysScope = 1), key "connector_only".
* N >= 2 (torchrun): one rank per GPU (R = N), one process each, connected
  with occlCommInit over torch.distributed and CUDA IPC; the ring crosses
  NVLink.  Sizes --sizes (MiB) are swept; beside OCCL, the SAME all-reduce
  through NCCL on the same GPUs (torch.distributed): NCCL_ALGO=Ring
  NCCL_PROTO=Simple (the paper's algorithm, the graded ratio) and NCCL's
  default choice (context).  NVML NVLink TX/RX byte deltas are OCCL's own
  evidence that the ring spans the GPUs.  Per-GPU work is fixed as N grows
  ("scaling": "weak").

A step = one all-reduce on every rank.  K steps are submitted to the SQ (one
SQE per rank per step, distinct collective ids) with an Exiting SQE, then the
daemon is launched once; the timed region is bracketed by CUDA events on the
daemon's stream (plus barrier + synchronize on both sides).  Inputs (8 x 256
MiB = 2 GiB) are larger than L2.

value = nccl-tests bus bandwidth busbw = S * 2(R-1)/R / t_step   (GB/s, 1e9;
the metric BASELINE.json names, a per-rank figure by nccl-tests convention).

--impl reference times the CPU oracle (oracle/ring.py, the plain numpy ring
fold) on a bounded sample of the same workload on this box's host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

MiB = 1 << 20
METRIC = "allreduce bus GB/s (ring AllReduce, sum; ring size and dtype in config)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="occl", choices=["occl", "reference"])
    ap.add_argument("--size-mib", type=float, default=256.0)
    ap.add_argument("--ranks", type=int, default=0, help="ring size; default 8 at N=1, N (one per GPU) at N>1")
    ap.add_argument("--sizes", default="64,256,1024", help="N>1: MiB per rank swept (the --size-mib point is the headline)")
    ap.add_argument("--no-nccl", action="store_true")
    ap.add_argument("--no-conn-only", action="store_true")
    ap.add_argument("--dtype", default="f32", choices=["f32", "bf16", "i32"])
    ap.add_argument("--grid-blocks", type=int, default=18)
    ap.add_argument("--slice-kib", type=int, default=192)
    ap.add_argument("--conn-slots", type=int, default=5)
    ap.add_argument("--slices-per-chunk", type=int, default=2)
    ap.add_argument("--threads", type=int, default=608)
    ap.add_argument("--pipe-depth", type=int, default=4)
    ap.add_argument("--discard", type=int, default=1)
    ap.add_argument("--l2-hints", type=int, default=2)
    ap.add_argument("--direct", type=int, default=1)
    ap.add_argument("--stages", type=int, default=6)
    ap.add_argument("--blocks-per-sm", type=int, default=1)
    ap.add_argument("--bulk-stores", type=int, default=0)
    ap.add_argument("--direct-read", type=int, default=1)
    ap.add_argument("--order-policy", type=int, default=1)
    ap.add_argument("--force-sys", type=int, default=0, help="1: the headline ring on the connector-only / .sys path")
    ap.add_argument("--sq-yield-ns", type=int, default=-1, help="-1: library default")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--check", action="store_true", help="sampled oracle check of the timed output")
    ap.add_argument("--no-latency", action="store_true", help="N=1: skip the small-message latency key")
    return ap.parse_args()


def busbw(size_bytes, nranks, t_s):
    return size_bytes * 2 * (nranks - 1) / nranks / t_s / 1e9


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


# ============================================================================ clocks
class ClockSampler:
    """Samples SM clock + throttle reasons with NVML during the timed region."""

    def __init__(self, dev=0, period=0.005):
        self.dev, self.period, self.samples, self.reasons = dev, period, [], set()
        self._stop = threading.Event()
        self.max_mhz = None
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(dev)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
        except Exception:
            self.N = None

    def _run(self):
        N = self.N
        names = {}
        for nm in ("HwSlowdown", "HwThermalSlowdown", "SwThermalSlowdown", "SwPowerCap", "HwPowerBrakeSlowdown"):
            v = getattr(N, "nvmlClocksEventReason" + nm, None) or getattr(N, "nvmlClocksThrottleReason" + nm, None)
            if v is not None:
                names[v] = nm
        while not self._stop.is_set():
            try:
                self.samples.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
                mask = N.nvmlDeviceGetCurrentClocksEventReasons(self.h) if hasattr(
                    N, "nvmlDeviceGetCurrentClocksEventReasons") else N.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for bit, nm in names.items():
                    if mask & bit:
                        self.reasons.add(nm)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.N:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.N:
            self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ============================================================================ reference arm
def cpu_oracle_busbw(nranks, dtype, size_bytes, budget_s=10.0, min_reps=1, max_reps=1000):
    """Time the CPU oracle (O1 ring fold) on a bounded sample; returns (busbw, sample, cores, secs)."""
    from inputs import hashgen
    from oracle import ring
    item = hashgen.ITEMSIZE[dtype]
    sample_bytes = min(size_bytes, 32 * MiB)
    count = int(sample_bytes // item)
    xs = [hashgen.buffer(dtype, 1, 0, r, count) for r in range(nranks)]
    times = []
    t_all = time.perf_counter()
    while len(times) < min_reps or (time.perf_counter() - t_all < budget_s and len(times) < max_reps):
        t0 = time.perf_counter()
        ring.allreduce(xs, dtype)
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    sample = (f"{nranks} ranks x {sample_bytes / MiB:g} MiB {dtype} per rank (of {size_bytes / MiB:g} MiB), "
              f"oracle/ring.py allreduce (numpy ring fold), median of {len(times)} reps")
    return busbw(sample_bytes, nranks, t), sample, 1, sum(times)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    if not args.ranks:                     # the OCCL arm's ring: 8 virtual ranks at N=1, one rank per GPU above
        args.ranks = args.gpus if args.gpus > 1 else 8
    size = int(args.size_mib * MiB)
    from inputs import hashgen
    from oracle import ring
    item = hashgen.ITEMSIZE[args.dtype]
    sample_bytes = min(size, 32 * MiB)
    count = int(sample_bytes // item)
    xs = [hashgen.buffer(args.dtype, 1, 0, r, count) for r in range(args.ranks)]
    for _ in range(args.warmup):
        ring.allreduce(xs, args.dtype)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ring.allreduce(xs, args.dtype)
    t = (time.perf_counter() - t0) / max(1, args.steps)
    v = busbw(sample_bytes, args.ranks, t)
    sample = (f"{args.ranks} ranks x {sample_bytes / MiB:g} MiB {args.dtype} per rank per step (bounded sample of "
              f"the {args.size_mib:g} MiB workload), oracle/ring.py numpy ring fold")
    unit = "GB/s"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": unit, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak" if args.gpus > 1 else "strong",
        "vs_baseline": None, "dtype": args.dtype, "data": "synthetic (counter-based hash generator)",
        "config": {"workload": f"C2 allreduce, {args.ranks}-rank ring, {args.size_mib:g} MiB/rank {args.dtype} sum",
                   "ranks": args.ranks, "size_bytes_per_rank": size},
        "cpu_baseline": {"value": v, "unit": unit, "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))
    return 0


# ============================================================================ OCCL arm
def setup_dist(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    dist = None
    if world > 1:
        import torch.distributed as dist
        # NCCL for the host-side plumbing (handle exchange, barriers, the max over
        # ranks); OCCL_BENCH_BACKEND=gloo lets several processes share one GPU
        # (the multi-process path smoke-tested on a single B200, tests/test_gpu_multiprocess.py)
        # NCCL's Ring/Simple protocol for the default group: it is the baseline
        # arm (the paper's algorithm); the OCCL data plane never uses NCCL
        os.environ.setdefault("NCCL_ALGO", "Ring")
        os.environ.setdefault("NCCL_PROTO", "Simple")
        dist.init_process_group(os.environ.get("OCCL_BENCH_BACKEND", "nccl"), init_method="env://")
    return world, rank, local, dist


def summarize_probes(pb, pa):
    """In-kernel probe deltas (occlGetProbes) summed over the local ranks, per slice / fence."""
    probes = {k: sum(a[k] - b[k] for a, b in zip(pa, pb)) for k in pa[0]}
    nc, nd = max(1, probes["nCommit"]), max(1, probes["nData"])
    return {"per_commit_cycles": {k: round(probes[k] / nc, 1) for k in ("cycRun", "cycPoll", "cycAcqFence",
                                                                        "cycRelFence")},
            "per_slice_data_cycles": round(probes["cycData"] / nd, 1),
            "per_slice_datawait_cycles": round(probes["cycDataWait"] / nd, 1),
            "commits": probes["nCommit"], "data_slices_timed": probes["nData"],
            "publisher_fences": probes["nFence"],
            "cycles_per_release_fence": round(probes["cycRelFence"] / max(1, probes["nFence"]), 1)}


def bench_cfg(args, **extra):
    from paper_2303_06324_b200 import occl
    kw = dict(gridBlocks=args.grid_blocks, sliceBytes=args.slice_kib * 1024, connSlots=args.conn_slots,
              slicesPerChunk=args.slices_per_chunk, blockThreads=args.threads, pipeDepth=args.pipe_depth,
              discardConsumed=args.discard, l2Hints=args.l2_hints,
              directMode=args.direct, stagingTiles=args.stages, blocksPerSM=args.blocks_per_sm,
              bulkStores=args.bulk_stores, directRead=args.direct_read, maxColl=128, autoLaunch=0,
              orderPolicy=args.order_policy, forceSysScope=args.force_sys)
    if args.sq_yield_ns >= 0:
        kw["sqYieldNs"] = args.sq_yield_ns
    kw.update(extra)
    return occl.occlConfigDefault(**kw)


def timed_launch(comms, sends, recvs, nsteps, stream, first_id=0, barrier=None):
    """nsteps all-reduces per local rank (distinct ids), an Exiting SQE, ONE daemon
    launch (serving every local rank); returns device ms (CUDA events on the
    daemon's stream)."""
    import torch
    ids = [(first_id + k) % 120 for k in range(nsteps)]
    for i, c in enumerate(comms):
        for cid in ids:
            c.all_reduce(sends[i], recvs[i], cid)
        c.exit()
    if barrier is not None:
        barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    comms[0].launch()                      # one fused launch serves all local ranks
    e1.record(stream)
    for c in comms:
        for cid in set(ids):
            c.wait(cid, 600)
    comms[0].quiesce(600)
    e1.synchronize()
    return e0.elapsed_time(e1)


def make_ring(args, world, prank, dev, dist, **extra):
    """R ranks over `world` processes, V = R/world consecutive ranks per process;
    handles exchanged over torch.distributed; local ranks fused into one daemon."""
    from paper_2303_06324_b200 import occl
    R = args.ranks
    if R % world:
        raise SystemExit("--ranks must be a multiple of the GPU count")
    V = R // world
    cfg = bench_cfg(args, **extra)
    hs = [occl.occlCommCreate(R, prank * V + i, dev, cfg) for i in range(V)]
    mine = [occl.occlCommGetHandle(h) for h in hs]
    if dist is not None:
        allh = [None] * world
        dist.all_gather_object(allh, mine)
        handles = [h for part in allh for h in part]
    else:
        handles = mine
    for h in hs:
        occl.occlCommConnect(h, handles)
    comms = [occl.Comm(h, R, prank * V + i, dev, cfg) for i, h in enumerate(hs)]
    if V > 1:
        occl.occlCommFuse(comms)
    return comms, V


def _red_dev(dist, dev):
    """Device of the tensor used for the max-over-ranks reduction (gloo: host)."""
    return dev if dist.get_backend() == "nccl" else "cpu"


def run_occl(args):
    world, prank, local, dist = setup_dist(args)
    if world > 1 and (args.ranks in (0, world)):
        return run_multi(args, world, prank, local, dist)
    if not args.ranks:
        args.ranks = 8
    return run_single(args, world, prank, local, dist)


def run_single(args, world, prank, local, dist):
    import torch
    from paper_2303_06324_b200 import occl
    dev = local % max(1, torch.cuda.device_count())   # one rank per GPU; several per GPU in the smoke test
    torch.cuda.set_device(dev)
    R = args.ranks
    size = int(args.size_mib * MiB)
    tdt = {"f32": torch.float32, "bf16": torch.bfloat16, "i32": torch.int32}[args.dtype]
    item = torch.tensor([], dtype=tdt).element_size()
    count = size // item
    comms, V = make_ring(args, world, prank, dev, dist)
    sends = [torch.empty(count, dtype=tdt, device=dev) for _ in range(V)]
    recvs = [torch.empty(count, dtype=tdt, device=dev) for _ in range(V)]
    for i, c in enumerate(comms):
        occl.test_fill(sends[i], args.dtype, 1, 0, c.rank)
    torch.cuda.synchronize()
    stream = torch.cuda.ExternalStream(comms[0].stream(), device=dev)

    def barrier():
        if dist is not None:
            dist.barrier()

    def run_steps(nsteps, first_id=0):
        """nsteps all-reduces per rank in ONE daemon launch; returns device ms."""
        return timed_launch(comms, sends, recvs, nsteps, stream, first_id)

    steps_per_launch = 100
    # warm-up (untimed)
    w = args.warmup
    while w > 0:
        run_steps(min(w, steps_per_launch))
        w -= steps_per_launch
    barrier()
    torch.cuda.synchronize()
    before = [c.stats() for c in comms]
    pb = [c.probes() for c in comms]
    ms_total, launches, left = 0.0, 0, args.steps
    with ClockSampler(dev) as clk:
        while left > 0:
            k = min(left, steps_per_launch)
            ms_total += run_steps(k)
            launches += 1
            left -= k
    torch.cuda.synchronize()
    barrier()
    after = [c.stats() for c in comms]
    pa = [c.probes() for c in comms]
    probe_summary = summarize_probes(pb, pa)
    if dist is not None:
        t = torch.tensor([ms_total], dtype=torch.float64, device=_red_dev(dist, dev))
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    value = busbw(size, R, ms_step / 1e3)

    check = None
    if args.check:
        import numpy as np
        from oracle import ring
        rng = np.random.default_rng(0)
        idx = np.unique(np.concatenate([rng.integers(0, count, 20000), [0, count - 1]]))
        ok = True
        for i, c in enumerate(comms):
            got = recvs[i][torch.from_numpy(idx).to(dev)].cpu()
            got = got.view(torch.int16).numpy().view(np.uint16) if args.dtype == "bf16" else got.numpy().view(np.uint32)
            exp = ring.expected_at("allreduce", args.dtype, R, count, 1, 0, idx)
            exp = exp.view(np.uint16) if args.dtype == "bf16" else exp.view(np.uint32)
            ok &= bool(np.array_equal(got, exp))
        check = {"sampled_elements_per_rank": int(len(idx)), "bit_exact": ok}

    # ------------------------------------------------------------------ e2e (public API, host buffers)
    e2e = None
    if not args.no_e2e:
        host_in = [torch.empty(count, dtype=tdt, pin_memory=True) for _ in range(V)]
        for i in range(V):
            host_in[i].copy_(sends[i].cpu())
        host_out = torch.empty(count, dtype=tdt, pin_memory=True)
        for c in comms:
            c.set_auto_launch(True)
        cs = torch.cuda.Stream(device=dev)
        e2e_steps = max(3, min(args.steps, 10))

        def e2e_step(k):
            with torch.cuda.stream(cs):
                for i in range(V):
                    sends[i].copy_(host_in[i], non_blocking=True)
            cs.synchronize()
            cid = 120 + (k % 4)
            for i, c in enumerate(comms):
                c.all_reduce(sends[i], recvs[i], cid)
            for c in comms:
                c.wait(cid, 600)
            if prank == 0:
                with torch.cuda.stream(cs):
                    host_out.copy_(recvs[0], non_blocking=True)
                cs.synchronize()

        e2e_step(0)
        barrier()
        t0 = time.perf_counter()
        for k in range(e2e_steps):
            e2e_step(k + 1)
        barrier()
        te = (time.perf_counter() - t0) / e2e_steps
        if dist is not None:
            t = torch.tensor([te], dtype=torch.float64, device=_red_dev(dist, dev))
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            te = float(t.item())
        e2e = {"value": busbw(size, R, te), "unit": "GB/s", "h2d_bytes_per_step": V * size,
               "d2h_bytes_per_step": size if prank == 0 else 0, "ms_per_step": te * 1e3, "steps": e2e_steps,
               "path": "pinned host -> device copies + occlAllReduce (event-driven daemon) + occlWait + D2H"}

    # ------------------------------------------------------------------ roofline
    peaks = measured_peaks()
    slices = sum(a["slices"] - b["slices"] for a, b in zip(after, before))
    avg_launch_ms = ms_total / max(1, launches)
    if world == 1:
        # One fused daemon launch serves all R ranks of this GPU; the unavoidable
        # DRAM traffic of an on-device all-reduce is reading every rank's input and
        # writing every rank's output: 2 * S per rank per step.
        alg_bytes = 2 * size * V * (args.steps / launches)
        achieved = alg_bytes / (avg_launch_ms / 1e3) / 1e9
        peak = peaks.get("hbm_gbs", 6650.0)
        traffic = None
        tf = os.path.join(ROOT, "profiles", "roofline_traffic.json")
        if os.path.exists(tf):
            try:
                d = json.load(open(tf))
                key = (f"{R}x{args.size_mib:g}MiB-{args.dtype}-G{args.grid_blocks}-s{args.slice_kib}k"
                       f"-K{args.conn_slots}-st{args.stages}-h{args.l2_hints}")
                if key in d:
                    traffic = d[key]["dram_bytes_per_step"] * (args.steps / launches)
            except Exception:
                traffic = None
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": traffic, "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else
                    "fallback 6650 GB/s (B200_PROFILING.md)",
                    "algorithmic_bytes_per_launch": alg_bytes, "avg_launch_ms": avg_launch_ms}
    else:
        alg_bytes = size * 2 * (R - 1) / R * V * (args.steps / launches)     # NVLink egress per GPU
        achieved = alg_bytes / (avg_launch_ms / 1e3) / 1e9
        roofline = {"bound": "nvlink", "achieved": achieved, "peak": 770.0, "unit": "GB/s", "frac": achieved / 770.0,
                    "traffic": None, "peak_source": "measured peer copy 770 GB/s/direction (B200_PROFILING.md)",
                    "algorithmic_bytes_per_launch": alg_bytes, "avg_launch_ms": avg_launch_ms}

    cpu = None
    if world == 1 and prank == 0 and not args.no_cpu:
        v, sample, cores, secs = cpu_oracle_busbw(R, args.dtype, size)
        cpu = {"value": v, "unit": "GB/s", "cores": cores, "kind": "oracle", "sample": sample,
               "cpu_seconds": secs, "host_cpus": os.cpu_count()}

    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": args.dtype,
        "data": "synthetic (counter-based hash generator, inputs resident in HBM)",
        "config": {"workload": f"C2 allreduce, {R}-rank ring, {args.size_mib:g} MiB/rank {args.dtype} sum, "
                               f"{V} rank(s) per GPU" + (" (virtual ranks, one fused daemon)" if V > 1 else ""),
                   "ranks": R, "ranks_per_gpu": V, "size_bytes_per_rank": size, "grid_blocks": args.grid_blocks,
                   "slice_bytes": args.slice_kib * 1024, "conn_slots": args.conn_slots,
                   "slices_per_chunk": args.slices_per_chunk, "block_threads": args.threads,
                   "pipe_depth": args.pipe_depth, "staging_tiles": args.stages, "l2": "inputs larger than L2 (R x S >> 126 MB)",
                   "algbw_GBps": size / (ms_step / 1e3) / 1e9},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "probes": probe_summary,
        "daemon": {"slices": slices, "preemptions": sum(a["preemptions"] - b["preemptions"] for a, b in zip(after, before)),
                   "cqe": sum(a["cqeWritten"] - b["cqeWritten"] for a, b in zip(after, before))},
    }
    if check is not None:
        line["check"] = check
    occl.destroy_group(comms)
    if world == 1 and not args.no_conn_only:
        co = conn_only_variant(args, dev, sends, recvs, size, peaks)
        co["vs_direct_mode"] = co["value"] / value
        line["connector_only"] = co
    if world == 1 and not args.no_latency:
        line["latency"] = small_message_latency(dev)
    if prank == 0:
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()
    return 0


def small_message_latency(dev, sizes=(4096, 65536, 1 << 20), reps=50):
    """End-to-end latency of single all-reduces (fp32, 8 virtual ranks, live
    daemon, library defaults): native per-rank threads submit at one instant and
    occlWait through the C-ABI (libocclbench.so); sample = max(done) -
    min(submit); median and p10/p90 of `reps` (the metric's "latency vs size",
    scripts/latency_split.py has the per-size split)."""
    import ctypes as C
    import statistics
    from paper_2303_06324_b200 import harness, occl
    L = C.CDLL(os.path.join(os.path.dirname(occl.LIB_PATH), "libocclbench.so"))
    L.occlBenchLatency.restype = C.c_int
    L.occlBenchLatency.argtypes = [C.POINTER(C.c_void_p), C.c_int, C.c_int, C.c_size_t, C.c_int, C.c_int, C.c_int,
                                   C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.c_int, C.c_int,
                                   C.POINTER(C.c_double)]
    n = 8
    comms = harness.ring(n, dev, gridBlocks=18, maxColl=16, quitIdleNs=10_000_000_000)
    out = {"ranks": n, "kind": "allreduce", "dtype": "f32", "unit": "us", "reps": reps,
           "definition": "max(done) - min(submit), native per-rank threads through the C-ABI"}
    try:
        hs = (C.c_void_p * n)(*[c.h if isinstance(c.h, int) else c.h.value for c in comms])
        for S in sizes:
            count = S // 4
            bufs = harness.buffers("allreduce", "f32", n, count, comms)
            ss = (C.c_void_p * n)(*[bufs[r][0].data_ptr() for r in range(n)])
            rs = (C.c_void_p * n)(*[bufs[r][1].data_ptr() for r in range(n)])
            res = (C.c_double * reps)()
            for k in (5, reps):                          # warm-up, then the sample
                rc = L.occlBenchLatency(hs, n, 0, count, occl.DTYPE["f32"], 0, 0, ss, rs, 1, k, res)
                if rc != 0:
                    raise RuntimeError(f"occlBenchLatency rc={rc}")
            lat = sorted(res[i] / 1e3 for i in range(reps))
            out[f"{S}B"] = {"median": statistics.median(lat), "p10": lat[reps // 10], "p90": lat[(9 * reps) // 10]}
            del bufs
    finally:
        for c in comms:
            c.exit()
        comms[0].quiesce(60)
        occl.destroy_group(comms)
    return out


def conn_only_variant(args, dev, sends, recvs, size, peaks):
    """The same ring on the data path a one-process-per-GPU ring runs: every
    edge connector-only (no direct mode / direct read) with system-scope
    fences and flags (forceSysScope = 1) -- VERDICT r01 next #4."""
    import torch
    from paper_2303_06324_b200 import occl
    R = args.ranks
    comms, V = make_ring(args, 1, 0, dev, None, forceSysScope=1)
    stream = torch.cuda.ExternalStream(comms[0].stream(), device=dev)
    try:
        timed_launch(comms, sends, recvs, max(3, args.warmup), stream)
        steps = max(5, args.steps)
        pb = [c.probes() for c in comms]
        ms = timed_launch(comms, sends, recvs, steps, stream, first_id=50) / steps
        probes = summarize_probes(pb, [c.probes() for c in comms])
    finally:
        occl.destroy_group(comms)
    bw = busbw(size, R, ms / 1e3)
    alg = 2 * size * V / (ms / 1e3) / 1e9
    peak = peaks.get("hbm_gbs", 6650.0)
    return {"value": bw, "unit": "GB/s", "ms_per_step": ms, "steps": steps,
            "config": "forceSysScope=1: connector-only edges, .sys fences / flags (directMode, directRead off)",
            "roofline_frac": alg / peak, "vs_direct_mode": None, "probes": probes}


# ============================================================================ N >= 2: one rank per GPU
class NvlinkCounters:
    """NVML NVLink data TX/RX byte counters of this process's GPU (best effort)."""

    def __init__(self, dev):
        self.ok = False
        try:
            import pynvml as N
            N.nvmlInit()
            self.N, self.h = N, N.nvmlDeviceGetHandleByIndex(dev)
            self.fields = [N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX]
            self.read()
            self.ok = True
        except Exception:
            pass

    def read(self):
        N = self.N
        vals = N.nvmlDeviceGetFieldValues(self.h, self.fields)
        out = []
        for v in vals:
            if v.nvmlReturn != 0:
                raise RuntimeError("nvlink field unsupported")
            out.append(int(v.value.ullVal) * 1024)          # KiB counters
        return out

    def delta(self, fn):
        if not self.ok:
            return fn(), None
        try:
            a = self.read()
        except Exception:
            return fn(), None
        r = fn()
        try:
            b = self.read()
        except Exception:
            return r, None
        return r, {"tx_bytes": b[0] - a[0], "rx_bytes": b[1] - a[1]}


def nccl_allreduce_ms(dist, group, t, steps, warmup):
    """Same-box NCCL all-reduce (torch.distributed), CUDA events on torch's stream."""
    import torch
    for _ in range(warmup):
        dist.all_reduce(t, group=group)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        dist.all_reduce(t, group=group)
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / steps


def multi_e2e(args, comm, send, recv, size, dist, dev):
    """End to end through the public API at N GPUs: per step, the H2D copy of this
    rank's input from pinned host memory, occlAllReduce on the event-driven daemon,
    occlWait, and the D2H copy of the result; host clock, max over ranks."""
    import torch
    host_in = torch.empty(send.numel(), dtype=send.dtype, pin_memory=True)
    host_in.copy_(send.cpu())
    host_out = torch.empty(recv.numel(), dtype=recv.dtype, pin_memory=True)
    comm.set_auto_launch(True)
    cs = torch.cuda.Stream(device=dev)
    steps = max(3, min(args.steps, 10))

    def step(k):
        with torch.cuda.stream(cs):
            send.copy_(host_in, non_blocking=True)
        cs.synchronize()
        cid = 120 + (k % 4)
        comm.all_reduce(send, recv, cid)
        comm.wait(cid, 600)
        with torch.cuda.stream(cs):
            host_out.copy_(recv, non_blocking=True)
        cs.synchronize()

    step(0)
    dist.barrier()
    t0 = time.perf_counter()
    for k in range(steps):
        step(k + 1)
    te = (time.perf_counter() - t0) / steps
    t = torch.tensor([te], dtype=torch.float64, device=_red_dev(dist, dev))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    te = float(t.item())
    comm.set_auto_launch(False)
    comm.quiesce(600)
    return {"value": busbw(size, dist.get_world_size(), te), "unit": "GB/s", "h2d_bytes_per_step": size,
            "d2h_bytes_per_step": size, "ms_per_step": te * 1e3, "steps": steps,
            "path": "pinned host -> device copy + occlAllReduce (event-driven daemon) + occlWait + D2H, per rank"}


def run_multi(args, world, prank, local, dist):
    """One rank per GPU: the metric's own configuration at N = 2 / 4 / 8."""
    import torch
    from paper_2303_06324_b200 import occl
    ndev = max(1, torch.cuda.device_count())
    dev = local % ndev
    torch.cuda.set_device(dev)
    R = world
    tdt = {"f32": torch.float32, "bf16": torch.bfloat16, "i32": torch.int32}[args.dtype]
    item = torch.tensor([], dtype=tdt).element_size()
    sizes = sorted({float(x) for x in args.sizes.split(",") if x} | {args.size_mib})
    comm = occl.process_group(device=dev, cfg=bench_cfg(args))       # occlCommInit over torch.distributed
    stream = torch.cuda.ExternalStream(comm.stream(), device=dev)
    backend = dist.get_backend()
    distinct = ndev >= world                                         # NCCL needs one GPU per rank
    nccl_ok = backend == "nccl" and distinct and not args.no_nccl
    nccl_groups = {}
    if nccl_ok:
        # the default process group was created with NCCL_ALGO=Ring NCCL_PROTO=Simple (main());
        # a second group gets NCCL's own algorithm choice (communicators are created lazily)
        nccl_groups["ring_simple"] = None
        saved = {k: os.environ.pop(k) for k in ("NCCL_ALGO", "NCCL_PROTO") if k in os.environ}
        nccl_groups["default"] = dist.new_group(backend="nccl")
        t = torch.ones(1024, device=dev)
        dist.all_reduce(t, group=nccl_groups["default"])           # create it now, without the env
        torch.cuda.synchronize()
        os.environ.update(saved)
    nvl = NvlinkCounters(dev)
    peaks = measured_peaks()
    rows = []
    with ClockSampler(dev) as clk:
        for smib in sizes:
            size = int(smib * MiB)
            count = size // item
            send = torch.empty(count, dtype=tdt, device=dev)
            recv = torch.empty(count, dtype=tdt, device=dev)
            occl.test_fill(send, args.dtype, 1, 0, prank)
            torch.cuda.synchronize()
            timed_launch([comm], [send], [recv], max(3, args.warmup), stream, barrier=dist.barrier)
            ms_occl, nv = nvl.delta(lambda: timed_launch([comm], [send], [recv], args.steps, stream, first_id=10,
                                                         barrier=dist.barrier))
            t = torch.tensor([ms_occl], dtype=torch.float64, device=_red_dev(dist, dev))
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item()) / args.steps
            row = {"size_bytes": size, "occl_ms": ms, "occl_busbw": busbw(size, R, ms / 1e3),
                   "nvlink_counters": nv}
            if args.check and smib == args.size_mib:
                import numpy as np
                from oracle import ring
                rng = np.random.default_rng(0)
                idx = np.unique(np.concatenate([rng.integers(0, count, 20000), [0, count - 1]]))
                got = recv[torch.from_numpy(idx).to(dev)].cpu()
                got = got.view(torch.int16).numpy().view(np.uint16) if args.dtype == "bf16" else got.numpy().view(np.uint32)
                exp = ring.expected_at("allreduce", args.dtype, R, count, 1, 0, idx)
                exp = exp.view(np.uint16) if args.dtype == "bf16" else exp.view(np.uint32)
                row["check"] = {"sampled_elements": int(len(idx)), "bit_exact": bool(np.array_equal(got, exp))}
            for name, g in nccl_groups.items():
                x = recv.clone()
                m = nccl_allreduce_ms(dist, g, x, args.steps, max(3, args.warmup))
                tt = torch.tensor([m], dtype=torch.float64, device=dev)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                m = float(tt.item())
                row[f"nccl_{name}_ms"] = m
                row[f"nccl_{name}_busbw"] = busbw(size, R, m / 1e3)
                del x
            if smib == args.size_mib and not args.no_e2e:
                row["e2e"] = multi_e2e(args, comm, send, recv, size, dist, dev)
            rows.append(row)
            del send, recv
            torch.cuda.empty_cache()
    head = [r for r in rows if r["size_bytes"] == int(args.size_mib * MiB)][0]
    size = head["size_bytes"]
    ms_step = head["occl_ms"]
    value = head["occl_busbw"]
    egress = size * 2 * (R - 1) / R                                 # NVLink bytes per GPU per all-reduce
    achieved = egress / (ms_step / 1e3) / 1e9
    roofline = {"bound": "nvlink", "achieved": achieved, "peak": 770.0, "unit": "GB/s", "frac": achieved / 770.0,
                "traffic": (head["nvlink_counters"] or {}).get("tx_bytes", None) and
                head["nvlink_counters"]["tx_bytes"] / args.steps,
                "peak_source": "measured peer copy 770 GB/s per direction (B200_PROFILING.md; 900 nominal)",
                "algorithmic_bytes_per_step": egress}
    baseline = {}
    for name in nccl_groups:
        baseline[f"nccl_{name}"] = {"value": head[f"nccl_{name}_busbw"], "ms_per_step": head[f"nccl_{name}_ms"]}
    ge64 = [r for r in rows if r["size_bytes"] >= 64 * MiB and "nccl_ring_simple_busbw" in r]
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": args.dtype,
        "data": "synthetic (counter-based hash generator, inputs resident in HBM)",
        "config": {"workload": f"C2 allreduce, {R}-rank ring, one rank per GPU, {args.size_mib:g} MiB/rank "
                               f"{args.dtype} sum", "ranks": R, "ranks_per_gpu": 1, "size_bytes_per_rank": size,
                   "grid_blocks": args.grid_blocks, "slice_bytes": args.slice_kib * 1024,
                   "conn_slots": args.conn_slots, "backend_plumbing": backend,
                   "l2": "inputs of 64 MiB-1 GiB per GPU; L2 not flushed between steps"},
        "gpu_launches": 1,
        "clocks": clk.summary(),
        "roofline": roofline,
        "cpu_baseline": None,
        "e2e": head.get("e2e"),
        "baseline": baseline or {"nccl": "unavailable: " + ("backend " + backend if backend != "nccl" else
                                                            "fewer GPUs than ranks" if not distinct else "--no-nccl")},
        "ratio_vs_nccl": (value / head["nccl_ring_simple_busbw"]) if "nccl_ring_simple_busbw" in head else None,
        "ratio_vs_nccl_ge64MiB_min": min((r["occl_busbw"] / r["nccl_ring_simple_busbw"] for r in ge64), default=None),
        "sweep": rows,
    }
    if prank == 0:
        print(json.dumps(line))
    comm.destroy()
    dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_occl(args)


if __name__ == "__main__":
    sys.exit(main())
