#!/bin/bash
cd "$GRAFT_REPO_ROOT"
W=c3,resnet50-buckets,resnet50-tensors,bert-large-buckets
for rf in 2 1; do
  timeout 1200 python scripts/live_c3_c4.py --seeds 2 --repeats 1 --iterations 20 --workloads $W --variants priority --ready-first $rf --tag "rf$rf" --out gpurun_out/m18_live_rf$rf > gpurun_out/m18_live_rf$rf.log 2>&1; echo "rf$rf rc=$?"
  grep SUMMARY gpurun_out/m18_live_rf$rf.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l[8:]); print('  ', d['workload'], 'cons', round(d['ms_consistent_median'],2), 'rand', round(d['ms_random_median'],2), 'vs ideal rand', round(d['overhead_vs_ideal_random_median'],3), 'cons', round(d['overhead_vs_ideal_consistent_median'],3), 'pre', d['preempt_random_median'])"
done
OCCL_RF=2 timeout 900 python -m pytest tests/test_gpu_sched.py tests/test_gpu_live.py -q --timeout 600 -p no:cacheprovider > gpurun_out/m18_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/m18_tests.log
