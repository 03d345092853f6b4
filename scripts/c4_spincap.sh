for cap in 65536 8192; do
python - <<PY
import sys, json
sys.path.insert(0, '.'); sys.path.insert(0, 'scripts')
import torch
from inputs import workloads
from paper_2303_06324_b200 import harness, occl
import mixed_c3 as M
n = 8
for wname in ("resnet50-tensors", "c3"):
    for stick in (1, 0):
        comms = harness.ring(n, 0, gridBlocks=18, maxColl=256, autoLaunch=0, stickiness=stick, orderPolicy=1, spinCap=$cap)
        colls, orders = M.workload(wname, n, 0)
        bufs = {c.coll_id: harness.buffers(c.kind, c.dtype, n, c.count, comms) for c in colls}
        consistent = [sorted(range(len(colls)))] * n
        ms_c, st_c = M.run_variant(comms, colls, consistent, bufs)
        ms_r, st_r = M.run_variant(comms, colls, orders, bufs)
        print("cap", $cap, wname, "stick", stick, round(ms_c, 2), round(ms_r, 2), st_c["preemptions"], st_r["preemptions"], flush=True)
        occl.destroy_group(comms)
        del bufs; torch.cuda.empty_cache()
PY
done
