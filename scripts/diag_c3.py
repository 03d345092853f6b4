import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import torch
from inputs import workloads
from paper_2303_06324_b200 import harness, occl
n = 8
stick = int(os.environ.get("STICK", "1"))
comms = harness.ring(n, 0, gridBlocks=18, maxColl=256, autoLaunch=0, stickiness=stick, orderPolicy=1)
colls, orders = workloads.c3(n, 64, 0)
bufs = {c.coll_id: harness.buffers(c.kind, c.dtype, n, c.count, comms) for c in colls}
jobs = [(c.coll_id, c.kind, c.dtype, c.count, c.root, bufs[c.coll_id]) for c in colls]
ms = harness.timed_batch(comms, jobs, [sorted(range(64))] * n)
print("ms", ms)
rows = []
for c in colls:
    st = [cm.coll_stats(c.coll_id) for cm in comms]
    pre = sum(s["preemptions"] for s in st)
    nb = comms[0].coll_blocks(c.kind, c.count, c.dtype)
    rows.append((pre, c.coll_id, c.kind, c.dtype, c.count, nb, [s["preemptions"] for s in st]))
for r in sorted(rows, reverse=True)[:25]:
    print(r)
print("probes", [cm.probes() for cm in comms][0])
