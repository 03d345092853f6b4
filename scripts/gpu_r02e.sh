#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 1200 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_sched.py tests/test_gpu_live.py -q --timeout 600 -p no:cacheprovider > gpurun_out/r02e_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02e_tests.log
timeout 120 python scripts/probe_multicast.py > gpurun_out/r02e_multicast.json 2>&1; echo "probe rc=$?"; tail -2 gpurun_out/r02e_multicast.json
W=c3,resnet50-buckets,bert-large-buckets
COMMON="--seeds 2 --repeats 1 --iterations 10 --workloads $W --variants priority"
i=0
for knobs in "--spin-cap 65536" "--spin-cap 4096" "--spin-base 512 --spin-step 64 --spin-min 32 --spin-cap 1024"; do
  i=$((i+1))
  timeout 900 python scripts/live_c3_c4.py $COMMON $knobs --tag "y$i: sqyield $knobs" --out gpurun_out/r02e_live_y$i > gpurun_out/r02e_live_y$i.log 2>&1; echo "y$i rc=$?"
  grep SUMMARY gpurun_out/r02e_live_y$i.log | cut -c1-300
done
for cq in 0 1 2; do
  timeout 900 python scripts/latency_split.py --kinds allreduce --cq-mode $cq --tag cq$cq --out gpurun_out/r02e_lat_cq$cq > gpurun_out/r02e_lat_cq$cq.log 2>&1; echo "lat cq$cq rc=$?"
  python -c "
import json
for l in open('gpurun_out/r02e_lat_cq$cq.jsonl'):
    d=json.loads(l); s=d['split'] or {}
    print(d['kind'], d['bytes'], round(d['e2e_median_us'],1), round(d['e2e_p10_us'],1), round(d['cqe_write_us'],2), {k:(round(v,2) if isinstance(v,float) else v) for k,v in s.items()})
"
done
bash scripts/gpu_traffic.sh
