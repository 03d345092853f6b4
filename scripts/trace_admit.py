#!/usr/bin/env python
"""Where "parse + load" goes for a small collective: native per-rank threads
submit at one instant (libocclbench.so); the device trace of every rank's
lane-0 block gives, per sample, each rank's admission of the SQE (fetch event)
and switch-in, relative to the earliest admission.  Prints medians over samples
of: admission spread (last - first rank), last admission -> rank's switch-in."""
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bytes", type=int, default=4096)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default="gpurun_out/trace_admit.json")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    n, G = 8, 18
    L = C.CDLL(os.path.join(os.path.dirname(occl.LIB_PATH), "libocclbench.so"))
    L.occlBenchLatency.restype = C.c_int
    L.occlBenchLatency.argtypes = [C.POINTER(C.c_void_p), C.c_int, C.c_int, C.c_size_t, C.c_int, C.c_int, C.c_int,
                                   C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.c_int, C.c_int,
                                   C.POINTER(C.c_double)]
    comms = harness.ring(n, 0, gridBlocks=G, maxColl=16, traceCap=1 << 16, quitIdleNs=10_000_000_000)
    count = a.bytes // 4
    bufs = harness.buffers("allreduce", "f32", n, count, comms)
    cid = 1
    hs = (C.c_void_p * n)(*[c.h if isinstance(c.h, int) else c.h.value for c in comms])
    ss = (C.c_void_p * n)(*[bufs[r][0].data_ptr() for r in range(n)])
    rs = (C.c_void_p * n)(*[bufs[r][1].data_ptr() for r in range(n)])
    res = (C.c_double * a.reps)()
    try:
        L.occlBenchLatency(hs, n, 0, count, occl.DTYPE["f32"], 0, 0, ss, rs, cid, a.reps, res)
        e2e = sorted(res[i] / 1e3 for i in range(a.reps))
        b0 = cid % G
        tr = [comms[r].trace(b0) for r in range(n)]
        fetch = [[t for t, e, c, x in ev if e == "fetch" and c == cid] for ev in tr]
        sw = [[t for t, e, c, x in ev if e == "switch_in" and c == cid] for ev in tr]
        dn = [[t for t, e, c, x in ev if e == "done" and c == cid] for ev in tr]
        cq = [[t for t, e, c, x in ev if e == "cqe" and c == cid] for ev in tr]
        k = min(len(f) for f in fetch)
        spread, last_to_sw, sw_to_done, done_to_cqe, first_sw_spread = [], [], [], [], []
        own_admit_to_sw, others_after_last, mirror_to_admit = [], [], []
        # every block's "mirror written" marks (mark 4) per rank
        tr4 = []
        for r in range(n):
            ev4 = []
            for bb in range(G):
                ev4 += [(t, e, c, x) for t, e, c, x in comms[r].trace(bb) if e == "mark" and x == 4]
            tr4.append(ev4)
        for j in range(max(0, k - a.reps), k):
            fs = [fetch[r][j] for r in range(n)]
            # first switch-in of this sample on each rank
            sws = [min(t for t in sw[r] if t >= fetch[r][j]) for r in range(n)]
            dns = [min(t for t in dn[r] if t >= sws[r]) for r in range(n)]
            spread.append((max(fs) - min(fs)) / 1e3)
            last = max(range(n), key=lambda r: fs[r])
            own_admit_to_sw.append((sws[last] - fs[last]) / 1e3)
            others_after_last.append(max((sws[r] - fs[last]) / 1e3 for r in range(n) if r != last))
            # the fetching block's mirror publish (mark 4) of the last rank, before its admission
            m4 = [t for t, e, c, x in tr4[last] if t <= fs[last]]
            if m4:
                mirror_to_admit.append((fs[last] - max(m4)) / 1e3)
            last_to_sw.append((max(sws) - max(fs)) / 1e3)
            first_sw_spread.append((max(sws) - min(sws)) / 1e3)
            sw_to_done.append((max(dns) - max(sws)) / 1e3)
        med = lambda v: round(statistics.median(v), 2)
        out = {"bytes": a.bytes, "e2e_median_us": med(e2e), "samples": len(spread),
               "admission_spread_us": med(spread), "last_admission_to_last_switch_in_us": med(last_to_sw),
               "switch_in_spread_us": med(first_sw_spread), "last_switch_in_to_last_done_us": med(sw_to_done),
               "last_admitter_admit_to_switch_in_us": med(own_admit_to_sw),
               "last_admission_to_others_switch_in_us": med(others_after_last),
               "last_admitter_mirror_to_admit_us": med(mirror_to_admit) if mirror_to_admit else None}
        print(json.dumps(out))
        with open(a.out, "w") as f:
            json.dump(out, f)
    finally:
        occl.destroy_group(comms)


if __name__ == "__main__":
    main()
