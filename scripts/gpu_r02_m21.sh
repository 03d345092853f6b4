#!/bin/bash
# Is the live path's overhead over the ideal schedule the voluntary quit / relaunch between buckets?
cd "$GRAFT_REPO_ROOT"
for q in 0 10000000; do
  timeout 1200 python scripts/live_c3_c4.py --seeds 2 --repeats 1 --iterations 20 --workloads resnet50-buckets,bert-large-buckets --variants priority --quit-idle-ns $q --tag "quit$q" --out gpurun_out/m21_q$q > gpurun_out/m21_q$q.log 2>&1; echo "quit $q rc=$?"
  grep SUMMARY gpurun_out/m21_q$q.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l[8:]); print('  ', d['tag'], d['workload'], 'cons', round(d['ms_consistent_median'],2), 'rand', round(d['ms_random_median'],2), 'vs ideal rand', round(d['overhead_vs_ideal_random_median'],3), 'cons', round(d['overhead_vs_ideal_consistent_median'],3), 'pre', d['preempt_random_median'])"
  python -c "
import json
for l in open('gpurun_out/m21_q$q.jsonl'):
    r=json.loads(l); print('    ', r['workload'][:10], r['seed'], 'launches', r['launches_random'], 'quits', r['quits_random'])"
done
timeout 900 python -m pytest tests/test_gpu_sched.py tests/test_gpu_subcomm.py -q --timeout 600 -p no:cacheprovider > gpurun_out/m21_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/m21_tests.log
