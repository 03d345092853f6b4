#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 1200 python scripts/live_c3_c4.py --seeds 2 --repeats 1 --iterations 20 --fifo-iterations 3 --fifo-seeds 1 --workloads c3,resnet50-buckets,resnet50-tensors,bert-large-buckets --variants priority,fifo+stickiness --out gpurun_out/m10_live > gpurun_out/m10_live.log 2>&1; echo "live rc=$?"; grep SUMMARY gpurun_out/m10_live.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l[8:]); print(d['workload'], d['variant'], 'cons', round(d['ms_consistent_median'],2), 'rand', round(d['ms_random_median'],2), 'ovh', round(d['overhead_median'],3), 'vs ideal rand', round(d['overhead_vs_ideal_random_median'],3), 'cons', round(d['overhead_vs_ideal_consistent_median'],3), 'pre', d['preempt_random_median'])"
