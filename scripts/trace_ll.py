#!/usr/bin/env python
"""Where a small (LL) all-reduce's hop goes, from the device trace: 8 virtual
ranks, one collective of --bytes (default 4 KiB, LL protocol, one block), the
daemon kept alive between samples.  Per hop (rank r step j+1 consuming rank
r-1's step j):
  detect  = issue(r, j+1) - sdone(r-1, j)   upstream's lines stored -> our control lane saw them
  move    = sdone(r, j+1) - issue(r, j+1)   descriptor -> compute warps polled, reduced, stored
and the per-collective split: first fetch -> first switch-in, switch-in -> done.
"""
import argparse
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2303_06324_b200 import harness, occl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bytes", type=int, default=4096)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--grid", type=int, default=18)
    ap.add_argument("--ll-max", type=int, default=-1)
    ap.add_argument("--ll-spec", type=int, default=0)
    ap.add_argument("--out", default="gpurun_out/trace_ll.json")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    n = 8
    extra = {"llMaxBytes": a.ll_max} if a.ll_max >= 0 else {}
    if a.ll_spec:
        extra["llSpeculate"] = 1
    comms = harness.ring(n, 0, gridBlocks=a.grid, maxColl=16, traceCap=1 << 14, quitIdleNs=10_000_000_000, **extra)
    cid = 1
    count = a.bytes // 4
    bufs = harness.buffers("allreduce", "f32", n, count, comms)
    det, mov, exe, adm = [], [], [], []
    parts = {k: [] for k in ("wake", "line_wait", "finish", "publish", "detect_from_store", "line_from_store",
                             "detect_from_last_store", "poll_start_to_last_store", "issue_to_next_poll_start",
                             "polled_late", "last_store_after_first", "run_slice_period", "run_start_to_done",
                             "run_stored_to_done", "run_upstream_stored_to_start")}
    try:
        for rep in range(a.reps):
            for c in comms:
                c.submit("allreduce", bufs[comms.index(c)][0], bufs[comms.index(c)][1], cid, count, "f32")
            for c in comms:
                c.wait(cid, 60)
            if rep < 3:
                continue
            b = cid % a.grid
            tr = [comms[r].trace(b) for r in range(n)]
            # this repetition's events only: after the last "fetch" of cid on each rank
            evs = []
            for r in range(n):
                f = max(i for i, (t, e, c, x) in enumerate(tr[r]) if e == "fetch" and c == cid)
                evs.append(tr[r][f:])
            issue = [[t for t, e, c, x in ev if e == "issue" and c == cid] for ev in evs]
            sdone = [[t for t, e, c, x in ev if e == "sdone"] for ev in evs]
            # LL runs (llSpeculate = 2): thread 0's marks per slice -- 40 start, 44 first line
            # in, 45 stores issued, 41 slice done (after the barrier and the credit)
            lr = {a: [[t for t, e, c, x in ev if e == "mark" and x == a] for ev in evs] for a in (40, 41, 44, 45)}
            for r in range(n):
                up = (r - 1) % n
                for j in range(1, len(lr[41][r])):
                    parts["run_slice_period"].append((lr[41][r][j] - lr[41][r][j - 1]) / 1e3)
                m = min(len(lr[40][r]), len(lr[41][r]), len(lr[45][r]))
                for j in range(m):
                    parts["run_start_to_done"].append((lr[41][r][j] - lr[40][r][j]) / 1e3)
                    parts["run_stored_to_done"].append((lr[41][r][j] - lr[45][r][j]) / 1e3)
                for j in range(1, min(len(lr[40][r]), len(lr[45][up]) + 1)):
                    parts["run_upstream_stored_to_start"].append((lr[40][r][j] - lr[45][up][j - 1]) / 1e3)
            # compute-warp marks of LL slices (20 woke, 21 first line in, 22 stored)
            mk = {a: [[t for t, e, c, x in ev if e == "mark" and x == a] for ev in evs] for a in (20, 21, 22, 23, 24)}
            # control lane: first failed poll of each slice (absent when the line was already there)
            for r in range(n):
                up = (r - 1) % n
                for j in range(1, min(len(issue[r]), len(mk[23][up]) + 1)):
                    parts["detect_from_last_store"].append((issue[r][j] - mk[23][up][j - 1]) / 1e3)
                    prev = issue[r][j - 1]
                    fp = [t for t, e, c, x in evs[r] if e == "mark" and x == 30 and prev < t <= issue[r][j]]
                    if fp:
                        parts["poll_start_to_last_store"].append((mk[23][up][j - 1] - fp[0]) / 1e3)
                        parts["issue_to_next_poll_start"].append((fp[0] - prev) / 1e3)
                    else:
                        parts["polled_late"].append(1.0)
                for j in range(min(len(mk[22][r]), len(mk[23][r]))):
                    parts["last_store_after_first"].append((mk[23][r][j] - mk[22][r][j]) / 1e3)
            for r in range(n):
                up = (r - 1) % n
                m = min(len(issue[r]), len(mk[20][r]), len(mk[21][r]), len(mk[22][r]), len(sdone[r]))
                for j in range(m):
                    parts["wake"].append((mk[20][r][j] - issue[r][j]) / 1e3)
                    if mk[21][r][j] > 0:
                        parts["line_wait"].append((mk[21][r][j] - mk[20][r][j]) / 1e3)
                        parts["finish"].append((mk[22][r][j] - mk[21][r][j]) / 1e3)
                    parts["publish"].append((sdone[r][j] - mk[22][r][j]) / 1e3)
                    if j >= 1 and j - 1 < len(mk[22][up]):
                        parts["detect_from_store"].append((issue[r][j] - mk[22][up][j - 1]) / 1e3)
                        if mk[21][r][j] > 0:
                            parts["line_from_store"].append((mk[21][r][j] - mk[22][up][j - 1]) / 1e3)
            for r in range(n):
                up = (r - 1) % n
                for j in range(1, min(len(issue[r]), len(sdone[up]) + 1)):
                    if j < len(issue[r]) and j - 1 < len(sdone[up]):
                        det.append((issue[r][j] - sdone[up][j - 1]) / 1e3)
                for j in range(min(len(issue[r]), len(sdone[r]))):
                    mov.append((sdone[r][j] - issue[r][j]) / 1e3)
                sw = [t for t, e, c, x in evs[r] if e == "switch_in" and c == cid]
                dn = [t for t, e, c, x in evs[r] if e == "done" and c == cid]
                if sw and dn:
                    exe.append((dn[-1] - sw[0]) / 1e3)
                    adm.append((sw[0] - evs[r][0][0]) / 1e3)
        # one sample's timeline on the lane-0 block of rank 0 and of rank 7: every
        # event from 30 us before the fetch of the last submission to its switch-in
        timeline = {}
        for rk in (0, n - 1):
            tr = comms[rk].trace(cid % a.grid)
            f = max(i for i, (t, e, c, x) in enumerate(tr) if e == "fetch" and c == cid)
            t0 = tr[f][0]
            sw = next((i for i in range(f, len(tr)) if tr[i][1] == "switch_in"), len(tr) - 1)
            timeline[rk] = [(round((t - t0) / 1e3, 2), e, c, x) for t, e, c, x in tr
                            if t0 - 30_000 <= t <= tr[sw][0]]
        # the same sample on every rank: fetch (admission), switch-in, done, CQE, relative
        # to the earliest admission (all ranks share %globaltimer)
        per_rank = {}
        for rk in range(n):
            tr = comms[rk].trace(cid % a.grid)
            f = max(i for i, (t, e, c, x) in enumerate(tr) if e == "fetch" and c == cid)
            ev = {}
            for t, e, c, x in tr[f:]:
                if e in ("fetch", "switch_in", "done", "cqe") and e not in ev:
                    ev[e] = t
            per_rank[rk] = ev
        tmin = min(v["fetch"] for v in per_rank.values())
        per_rank = {rk: {e: round((t - tmin) / 1e3, 2) for e, t in v.items()} for rk, v in per_rank.items()}
        # the full event sequence of one sample on rank 3's lane-0 block (switch-in .. done)
        tr3 = comms[3].trace(cid % a.grid)
        f = max(i for i, (t, e, c, x) in enumerate(tr3) if e == "fetch" and c == cid)
        t0 = tr3[f][0]
        run_seq = [(round((t - t0) / 1e3, 3), e, c, x) for t, e, c, x in tr3[f:]]
        res = {"run_sequence_rank3": run_seq, "bytes": a.bytes, "hops_sampled": len(det), "per_rank_last_sample_us": per_rank,
               "detect_us_median": statistics.median(det) if det else None,
               "detect_us_p10": sorted(det)[len(det) // 10] if det else None,
               "move_us_median": statistics.median(mov) if mov else None,
               "execute_us_median": statistics.median(exe) if exe else None,
               "fetch_to_switchin_us_median": statistics.median(adm) if adm else None,
               "issues_per_rank": len(issue[0]),
               "hop_parts_us_median": {k: (statistics.median(v) if v else None) for k, v in parts.items()},
               "hop_parts_n": {k: len(v) for k, v in parts.items()},
               "hop_parts_us_p10": {k: (sorted(v)[len(v) // 10] if v else None) for k, v in parts.items()},
               "timeline_lane0_block": timeline}
        print(json.dumps(res))
        with open(a.out, "w") as f:
            json.dump(res, f)
    finally:
        occl.destroy_group(comms)


if __name__ == "__main__":
    main()
