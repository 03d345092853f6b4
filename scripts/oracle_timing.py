#!/usr/bin/env python
"""The CPU oracle timed on the GPU box's host ("CPU oracle timed
beside the GPU").  Test infrastructure: it times oracle/ as it stands, untuned.

(i)   O1 numpy ring fold (oracle/ring.py allreduce) for C2 sizes 4 KiB..64 MiB,
      8 ranks, fp32, fully materialised, single core: "oracle GB/s" = n*S / t;
(ii)  O2 DFCE simulator (oracle/dfce.py) on C1 and on C3 scaled by 1/1024
      (8 ranks, 64 collectives): wall time and simulator ticks/s, single thread;
(iii) the brute-force order suite (every (k!)^n per-rank order set for
      n, k in {2, 3}) on all host cores via multiprocessing: wall time, cores.

Prints one JSON object; --out writes it too."""
import argparse
import itertools
import json
import multiprocessing as mp
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from inputs import hashgen, workloads  # noqa: E402
from oracle import dfce, ring  # noqa: E402


def _o1(max_bytes):
    rows = []
    n = 8
    S = 4096
    while S <= max_bytes:
        count = S // 4
        xs = [hashgen.buffer("f32", 1, 0, r, count) for r in range(n)]
        reps, t0 = 0, time.perf_counter()
        while True:
            ring.allreduce(xs, "f32")
            reps += 1
            dt = time.perf_counter() - t0
            if dt > 0.5 or reps >= 200:
                break
        rows.append({"bytes": S, "reps": reps, "s_per_op": dt / reps, "oracle_GBps": n * S / (dt / reps) / 1e9})
        S *= 4
    return rows


def _o2_run(metas, orders, cfg):
    t0 = time.perf_counter()
    sim, _ = dfce.run_orders(metas, orders, cfg, seed=3)
    dt = time.perf_counter() - t0
    return {"wall_s": dt, "ticks": sim.tick, "ticks_per_s": sim.tick / dt, "preemptions": sim.total_preemptions()}


def _o2():
    colls, orders = workloads.c1()
    c1 = _o2_run([dfce.CollMeta(c.coll_id, c.kind, c.dtype, c.count) for c in colls], orders,
                 dfce.SimConfig(spin_base=64, spin_step=4, spin_min=1, spin_cap=256, seed=1))
    colls, orders = workloads.c3(nranks=8, ncoll=64, seed=0, scale=1024)
    c3 = _o2_run([dfce.CollMeta(c.coll_id, c.kind, c.dtype, c.count, c.root) for c in colls], orders,
                 dfce.SimConfig(order_policy="priority", seed=1))
    return {"C1": c1, "C3_scaled_1_1024": c3}


_BF_CFG = dict(K=3, slice_elems=8, slices_per_chunk=2, quit_idle=64)


def _bf_one(args):
    n, k, si, orders = args
    sizes = [40, 96, 13]
    metas = [dfce.CollMeta(i, "allreduce", "f32", sizes[i % 3]) for i in range(k)]
    variants = [(T, st) for T in (1, 3, 64) for st in (False, True)]
    T, st = variants[si % len(variants)]
    cfg = dfce.SimConfig(spin_base=T, spin_step=max(1, T // 8), spin_min=1, spin_cap=4 * T, stickiness=st,
                         seed=si, **_BF_CFG)
    sim, bufs = dfce.run_orders(metas, [list(o) for o in orders], cfg, seed=si)
    # every output equals the O1 ring result (deadlock-free and exact)
    for m in metas:
        xs = [bufs[(r, m.coll_id, 0)][0] for r in range(n)]
        exp = ring.allreduce(xs, "f32")
        for r in range(n):
            if not np.array_equal(bufs[(r, m.coll_id, 0)][1], exp):
                return False
    return True


def _bruteforce():
    jobs = []
    for n, k in [(2, 2), (2, 3), (3, 2), (3, 3)]:
        perms = list(itertools.permutations(range(k)))
        for si, orders in enumerate(itertools.product(perms, repeat=n)):
            jobs.append((n, k, si, orders))
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(cores) as pool:
        ok = pool.map(_bf_one, jobs, chunksize=4)
    return {"order_sets": len(jobs), "all_exact": all(ok), "wall_s": time.perf_counter() - t0, "cores": cores}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-bytes", type=int, default=64 << 20)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    res = {"host": {"cpus": os.cpu_count(), "processor": platform.processor() or platform.machine()},
           "o1_ring_fold_8ranks_f32_single_core": _o1(a.max_bytes), "o2_dfce_single_thread": _o2(),
           "bruteforce_all_orders": _bruteforce()}
    try:
        with open("/proc/cpuinfo") as f:
            res["host"]["model"] = next((l.split(":", 1)[1].strip() for l in f if l.startswith("model name")), "")
    except OSError:
        pass
    s = json.dumps(res)
    print(s)
    if a.out:
        with open(a.out, "w") as f:
            f.write(s + "\n")


if __name__ == "__main__":
    main()
