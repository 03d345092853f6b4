#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python scripts/trace_live.py --runs 30 --policy 1 --out gpurun_out/m8_trace_live_p1.json > gpurun_out/m8_trace_live_p1.log 2>&1; echo "p1 rc=$?"; grep makespan gpurun_out/m8_trace_live_p1.log | python -c "
import sys,json; r=[json.loads(l) for l in sys.stdin]; ms=sorted(x['makespan_ms'] for x in r); print('makespans', [round(m,2) for m in ms])"
timeout 600 python scripts/stickiness_case.py --out gpurun_out/m8_stickiness_case > gpurun_out/m8_stickiness.log 2>&1; echo "stickiness rc=$?"; cut -c1-250 gpurun_out/m8_stickiness.log | tail -4
timeout 1200 python scripts/live_c3_c4.py --seeds 2 --repeats 1 --iterations 20 --workloads c3,resnet50-buckets,resnet50-tensors,bert-large-buckets --variants priority --out gpurun_out/m8_live > gpurun_out/m8_live.log 2>&1; echo "live rc=$?"; grep SUMMARY gpurun_out/m8_live.log | cut -c1-330
