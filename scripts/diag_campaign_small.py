import sys, time, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, 'tests'))
import torch
from inputs import workloads
from paper_2303_06324_b200 import occl
import test_gpu_sched as T
variant = eval(sys.argv[1]) if len(sys.argv) > 1 else {}
comms = occl.local_group(8, 0, **dict(T.BASE, maxColl=16, **variant))
ts = []
for trial in range(int(os.environ.get("TRIALS", "6"))):
    colls, orders = workloads.deadlock_trial(8, 8, seed=trial)
    t0 = time.perf_counter()
    T._run_orders(comms, colls, orders, seed=trial, check=False)
    ts.append(round((time.perf_counter() - t0) * 1e3, 1))
    print(trial, ts[-1], flush=True)
st = comms[0].stats()
print(os.environ.get("OCCL_LIB_PATH"), variant, ts, {k: st[k] for k in ('launches', 'quits', 'preemptions', 'sqeFetched')}, flush=True)
occl.destroy_group(comms)
