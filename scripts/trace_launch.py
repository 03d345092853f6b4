"""Timeline of ONE small all-reduce in its own daemon launch (8 virtual ranks):
per rank, the first block start, SQE fetch, first switch-in, completion, CQE
and the last exit, relative to the earliest block start (device trace)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2303_06324_b200 import harness, occl  # noqa: E402

n = 8
comms = harness.ring(n, 0, gridBlocks=18, maxColl=16, autoLaunch=0, traceCap=4096)
count = 1024
bufs = harness.buffers("allreduce", "f32", n, count, comms)
job = [(0, "allreduce", "f32", count, 0, bufs)]
for _ in range(3):
    harness.timed_batch(comms, job)
for c in comms:
    c.trace_reset()
ms = harness.timed_batch(comms, job)
tr = {(r, b): comms[r].trace(b) for r in range(n) for b in range(18)}
t0 = min(t[0][0] for t in tr.values() if t)
res = {"launch_ms": ms}
for r in range(n):
    evs = {}
    for b in range(18):
        for t, ev, c, a in tr[(r, b)]:
            evs.setdefault(ev, []).append((t - t0) / 1e3)
    res[f"rank{r}"] = {ev: [round(min(v), 1), round(max(v), 1), len(v)] for ev, v in sorted(evs.items())}
print(json.dumps(res, indent=0))
for b in range(18):                                   # the fetching block's marks (rank 0)
    ms_ = [((t - t0) / 1e3, ev, c, a) for t, ev, c, a in tr[(0, b)] if ev in ("mark", "start", "fetch")]
    if any(e[1] == "mark" for e in ms_):
        print("rank0 block", b, [(round(x, 2), ev, c, a) for x, ev, c, a in ms_])
occl.destroy_group(comms)
