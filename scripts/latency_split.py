#!/usr/bin/env python
"""End-to-end latency vs size on a LIVE daemon, and the paper's time split
(fig:time_split: read SQE / parse + load / execute / write CQE).

8 virtual ranks (one fused daemon kept alive between samples).  Per size:
  * e2e: libocclbench.so's native per-rank threads submit + occlWait through the
    C-ABI at the same instant; sample = max(done) - min(submit) (host clock);
    median / p10 / p90 of `reps` samples;
  * split: one more sample with the device event trace on -- on the block that
    runs the collective's lane 0 of rank 0:
      read SQE    = the fetching block's PCIe round trip that returned the SQE
                    (mark 1 -> mark 2, this block or the one holding the fetch lock),
      parse+load  = mirror written (mark 4) -> switch-in (admission, context load),
      execute     = switch-in -> done (the ring's hops),
      write CQE   = done -> CQE store issued (completion counter, fence.sys).
"""
import argparse
import ctypes as C
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2303_06324_b200 import harness, occl  # noqa: E402

KIND = {"allreduce": 0, "allgather": 1, "reducescatter": 2, "broadcast": 3}


def bench_lib():
    # the harness next to the product library in use (OCCL_LIB_PATH: an A/B build)
    L = C.CDLL(os.path.join(os.path.dirname(occl.LIB_PATH), "libocclbench.so"))
    L.occlBenchLatency.restype = C.c_int
    L.occlBenchLatency.argtypes = [C.POINTER(C.c_void_p), C.c_int, C.c_int, C.c_size_t, C.c_int, C.c_int, C.c_int,
                                   C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.c_int, C.c_int,
                                   C.POINTER(C.c_double)]
    return L


def native_latency(L, comms, kind, count, dtype, bufs, cid, reps):
    n = len(comms)
    hs = (C.c_void_p * n)(*[c.h if isinstance(c.h, int) else c.h.value for c in comms])
    ss = (C.c_void_p * n)(*[bufs[r][0].data_ptr() for r in range(n)])
    rs = (C.c_void_p * n)(*[bufs[r][1].data_ptr() for r in range(n)])
    out = (C.c_double * reps)()
    rc = L.occlBenchLatency(hs, n, KIND[kind], count, occl.DTYPE[dtype], 0, 0, ss, rs, cid, reps, out)
    if rc != 0:
        raise RuntimeError(f"occlBenchLatency rc={rc}")
    return [out[i] / 1e3 for i in range(reps)]


def split_from_trace(comms, cid, G):
    """Time split of the last sample of collective `cid` on rank 0's lane-0 block."""
    b0 = cid % G
    tr = {b: comms[0].trace(b) for b in range(G)}
    ev = tr[b0]
    dones = sorted(t for t, e, c, a in ev if e == "done" and c == cid)
    if not dones:
        return None
    t_done = dones[-1]
    t_prev = dones[-2] if len(dones) > 1 else 0
    sws = [t for t, e, c, a in ev if e == "switch_in" and c == cid and t_prev < t <= t_done]
    cqe = [t for t, e, c, a in ev if e == "cqe" and c == cid and t >= t_done]
    if not sws:
        return None
    t_sw = min(sws)
    # the fetch round trip that returned the SQE: the last mark(2, valid > 0) before the switch-in
    rt = []
    for b in range(G):
        marks = [(t, c, a) for t, e, c, a in tr[b] if e == "mark"]
        for i, (t, c, a) in enumerate(marks):
            if a == 2 and c > 0 and t_prev < t <= t_sw:
                start = [tt for tt, cc, aa in marks[:i] if aa == 1]
                mirror = [tt for tt, cc, aa in marks[i:] if aa == 4]
                if start and mirror:
                    rt.append((t, start[-1], mirror[0]))
    res = {"execute_us": (t_done - t_sw) / 1e3, "switch_ins": len(sws),
           "write_cqe_us": (min(cqe) - t_done) / 1e3 if cqe else None}
    if rt:
        t2, t1, t4 = max(rt)
        res.update(read_sqe_us=(t2 - t1) / 1e3, parse_load_us=(t_sw - t4) / 1e3)
    return res


def stop(comms):
    """Exiting SQE to every member; wait until the fused daemon is gone."""
    for c in comms:
        c.exit()
    comms[0].quiesce(60)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ranks", type=int, default=8)
    ap.add_argument("--kinds", default="allreduce,allgather,reducescatter,broadcast")
    ap.add_argument("--sizes", default="4096,16384,65536,262144,1048576,4194304,16777216,67108864")
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--grid", type=int, default=18)
    ap.add_argument("--ll-max", type=int, default=-1)
    ap.add_argument("--ll-slice", type=int, default=0)
    ap.add_argument("--min-block", type=int, default=0)
    ap.add_argument("--cq-mode", type=int, default=0)
    ap.add_argument("--ll-spec", type=int, default=-1, help="llSpeculate (0 per-slice LL, 1 speculation, 2 LL runs)")
    ap.add_argument("--tag", default="")
    ap.add_argument("--out", default="gpurun_out/latency_split")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    n = a.ranks
    extra = {}
    if a.ll_max >= 0:
        extra["llMaxBytes"] = a.ll_max
    if a.ll_slice:
        extra["llSliceBytes"] = a.ll_slice
    if a.min_block:
        extra["minBlockBytes"] = a.min_block
    if a.cq_mode:
        extra["cqMode"] = a.cq_mode
    if a.ll_spec >= 0:
        extra["llSpeculate"] = a.ll_spec
    L = bench_lib()
    rows = []
    # e2e samples without tracing; the split from a second, traced ring (the trace's
    # atomics would perturb the latency being measured)
    comms = harness.ring(n, 0, gridBlocks=a.grid, maxColl=16, quitIdleNs=10_000_000_000, **extra)
    traced = harness.ring(n, 0, gridBlocks=a.grid, maxColl=16, traceCap=1 << 16, quitIdleNs=10_000_000_000,
                          **extra)
    try:
        for kind in a.kinds.split(","):
            for S in [int(x) for x in a.sizes.split(",")]:
                count = S // 4 // (n if kind in ("allgather", "reducescatter") else 1)
                bufs = harness.buffers(kind, "f32", n, max(1, count), comms)
                cid = 1
                native_latency(L, comms, kind, count, "f32", bufs, cid, 5)          # warm-up (daemon live)
                p0 = comms[0].probes()
                lat = sorted(native_latency(L, comms, kind, count, "f32", bufs, cid, a.reps))
                stop(comms)                          # one persistent daemon on the GPU at a time
                p1 = comms[0].probes()
                ncqe = p1["nCqe"] - p0["nCqe"]
                cqe_cyc = (p1["cycCqe"] - p0["cycCqe"]) / max(1, ncqe)
                native_latency(L, traced, kind, count, "f32", bufs, cid, 3)
                sp = split_from_trace(traced, cid, a.grid)                          # last occurrence of cid
                stop(traced)
                row = {"tag": a.tag, "knobs": extra, "kind": kind, "bytes": S, "ranks": n,
                       "e2e_median_us": statistics.median(lat), "e2e_p10_us": lat[len(lat) // 10],
                       "e2e_p90_us": lat[(9 * len(lat)) // 10], "split": sp,
                       "cqe_write_cycles": cqe_cyc, "cqe_write_us": cqe_cyc / 1965.0, "cqes": ncqe}
                rows.append(row)
                print(json.dumps(row), flush=True)
                del bufs
    finally:
        occl.destroy_group(comms)
        occl.destroy_group(traced)
    with open(a.out + ".jsonl", "w") as f:
        for r in rows:
            f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
