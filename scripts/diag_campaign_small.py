"""Where does an event-driven (autoLaunch) trial of the small deadlock campaign
spend its time?  Per trial: wall time, launches, quits, preemptions, and the
largest idle gaps in the device traces."""
import sys, time, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, 'tests'))
import torch
from inputs import workloads
from paper_2303_06324_b200 import occl
import test_gpu_sched as T
variant = eval(sys.argv[1]) if len(sys.argv) > 1 else {}
comms = occl.local_group(8, 0, **dict(T.BASE, maxColl=16, traceCap=1 << 14, **variant))
prev = comms[0].stats()
for trial in range(int(os.environ.get("TRIALS", "6"))):
    colls, orders = workloads.deadlock_trial(8, 8, seed=trial)
    t0 = time.perf_counter()
    T._run_orders(comms, colls, orders, seed=trial, check=False)
    dt = (time.perf_counter() - t0) * 1e3
    st = comms[0].stats()
    d = {k: st[k] - prev[k] for k in ('launches', 'quits', 'preemptions', 'sqeFetched')}
    prev = st
    print(trial, round(dt, 1), d, flush=True)
comms[0].quiesce(60)
# biggest gaps between consecutive records of rank 0 block 0
tr = comms[0].trace(0)
gaps = sorted(((tr[i + 1][0] - tr[i][0]) / 1e3, tr[i][1:], tr[i + 1][1:]) for i in range(len(tr) - 1))[-12:]
for g in gaps:
    print("gap us %.1f after %s before %s" % g)
from collections import Counter
print(Counter(ev for _, ev, _, _ in tr))
occl.destroy_group(comms)
