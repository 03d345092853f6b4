#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 600 python scripts/trace_live.py --runs 30 --policy 1 --out gpurun_out/m6_trace_live_p1.json > gpurun_out/m6_trace_live_p1.log 2>&1; echo "p1 rc=$?"; grep makespan gpurun_out/m6_trace_live_p1.log | cut -c1-200
timeout 1200 python scripts/live_c3_c4.py --seeds 2 --repeats 1 --iterations 20 --fifo-iterations 3 --fifo-seeds 1 --workloads c3,resnet50-buckets,resnet50-tensors,bert-large-buckets --variants priority --out gpurun_out/m6_live > gpurun_out/m6_live.log 2>&1; echo "live rc=$?"; grep SUMMARY gpurun_out/m6_live.log | cut -c1-330
timeout 900 python -m pytest tests/test_gpu_sched.py tests/test_gpu_live.py tests/test_gpu_parity.py -q --timeout 600 -p no:cacheprovider > gpurun_out/m6_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/m6_tests.log
timeout 900 python scripts/latency_split.py --kinds allreduce --tag admitcache --out gpurun_out/m6_lat > gpurun_out/m6_lat.log 2>&1; echo "lat rc=$?"
python -c "
import json
for l in open('gpurun_out/m6_lat.jsonl'):
    d=json.loads(l); s=d['split'] or {}
    print(d['kind'][:6], d['bytes'], 'e2e med', round(d['e2e_median_us'],1), {k:(round(v,2) if isinstance(v,float) else v) for k,v in s.items()})"
