#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 1200 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_sched.py -q --timeout 600 -p no:cacheprovider > gpurun_out/r02d_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02d_tests.log
timeout 120 python scripts/probe_multicast.py > gpurun_out/r02d_multicast.json 2>&1; echo "probe rc=$?"; cat gpurun_out/r02d_multicast.json | tail -2
for cq in 0 1 2; do
  timeout 900 python scripts/latency_split.py --kinds allreduce --cq-mode $cq --tag cq$cq --out gpurun_out/r02d_lat_cq$cq > gpurun_out/r02d_lat_cq$cq.log 2>&1; echo "lat cq$cq rc=$?"
  python -c "
import json
for l in open('gpurun_out/r02d_lat_cq$cq.jsonl'):
    d=json.loads(l); s=d['split'] or {}
    print(d['kind'], d['bytes'], round(d['e2e_median_us'],1), round(d['e2e_p10_us'],1), round(d['cqe_write_us'],2), {k:(round(v,2) if isinstance(v,float) else v) for k,v in s.items()})
"
done
bash scripts/gpu_traffic.sh
