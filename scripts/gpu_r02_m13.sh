#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sched.py tests/test_gpu_subcomm.py tests/test_gpu_live.py tests/test_gpu_hazards.py tests/test_gpu_multiprocess.py -q --timeout 600 -p no:cacheprovider > gpurun_out/m13_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/m13_tests.log
W=c3,resnet50-buckets,resnet50-tensors,bert-large-buckets
for rf in 1 0; do
  timeout 1200 python scripts/live_c3_c4.py --seeds 2 --repeats 1 --iterations 20 --workloads $W --variants priority --ready-first $rf --tag "rf$rf" --out gpurun_out/m13_live_rf$rf > gpurun_out/m13_live_rf$rf.log 2>&1; echo "rf$rf rc=$?"
  grep SUMMARY gpurun_out/m13_live_rf$rf.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l[8:]); print('  ', d['workload'], 'cons', round(d['ms_consistent_median'],2), 'rand', round(d['ms_random_median'],2), 'vs ideal rand', round(d['overhead_vs_ideal_random_median'],3), 'cons', round(d['overhead_vs_ideal_consistent_median'],3), 'pre', d['preempt_random_median'])"
done
timeout 600 python scripts/stickiness_case.py --out gpurun_out/m13_stickiness_case > gpurun_out/m13_stickiness.log 2>&1; echo "stickiness rc=$?"; cut -c1-200 gpurun_out/m13_stickiness.log | tail -4
timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu --no-conn-only > gpurun_out/m13_bench.json 2>&1; echo "bench rc=$?"; cut -c1-200 gpurun_out/m13_bench.json
