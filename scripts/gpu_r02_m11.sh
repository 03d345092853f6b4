#!/bin/bash
cd "$GRAFT_REPO_ROOT"
W=c3,resnet50-buckets,bert-large-buckets
i=0
for knobs in "" "--spin-base 1024 --spin-step 64" "--spin-base 512 --spin-step 32 --spin-min 64" "--spin-base 2048 --spin-step 128 --spin-cap 16384"; do
  i=$((i+1))
  timeout 900 python scripts/live_c3_c4.py --seeds 2 --repeats 1 --iterations 20 --workloads $W --variants priority $knobs --tag "k$i $knobs" --out gpurun_out/m11_live_k$i > gpurun_out/m11_live_k$i.log 2>&1; echo "k$i [$knobs] rc=$?"
  grep SUMMARY gpurun_out/m11_live_k$i.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l[8:]); print('  ', d['workload'], 'cons', round(d['ms_consistent_median'],2), 'rand', round(d['ms_random_median'],2), 'vs ideal rand', round(d['overhead_vs_ideal_random_median'],3), 'cons', round(d['overhead_vs_ideal_consistent_median'],3), 'pre', d['preempt_random_median'])"
done
