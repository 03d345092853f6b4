"""FIFO + stickiness under independent random orders (C3): sensitivity to the
reading-dependent knobs (stall limit R3, threshold scale R1)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "scripts"))
import torch
from paper_2303_06324_b200 import harness, occl
import mixed_c3 as M
n = 8
for name, kw in [("default", {}), ("stall1", dict(stallLimit=1)), ("base512", dict(spinBase=512, spinStep=64, spinMin=16)),
                 ("stall1+base512", dict(stallLimit=1, spinBase=512, spinStep=64, spinMin=16))]:
    for stick in (1, 0):
        comms = harness.ring(n, 0, gridBlocks=18, maxColl=256, autoLaunch=0, stickiness=stick, orderPolicy=0, **kw)
        colls, orders = M.workload("c3", n, 0)
        bufs = {c.coll_id: harness.buffers(c.kind, c.dtype, n, c.count, comms) for c in colls}
        ms_r, st_r = M.run_variant(comms, colls, orders, bufs)
        print(json.dumps({"variant": name, "stickiness": stick, "ms_random": ms_r, "preemptions": st_r["preemptions"]}), flush=True)
        occl.destroy_group(comms)
        del bufs
        torch.cuda.empty_cache()
