#!/bin/bash
cd "$GRAFT_REPO_ROOT"
W=c3,resnet50-buckets,resnet50-tensors,bert-large-buckets
for pass in 1 2; do
OCCL_LIB_PATH=paper_2303_06324_b200/lib/exp/lib_scan8.so timeout 1200 python scripts/live_c3_c4.py --seeds 2 --repeats 1 --iterations 20 --workloads $W --variants priority --tag scan8 --out gpurun_out/m19_live_s8_p$pass > gpurun_out/m19_live_s8_p$pass.log 2>&1; echo "scan8 rc=$?"
grep SUMMARY gpurun_out/m19_live_s8_p$pass.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l[8:]); print('  s8', d['workload'], 'cons', round(d['ms_consistent_median'],2), 'rand', round(d['ms_random_median'],2), 'vs ideal rand', round(d['overhead_vs_ideal_random_median'],3), 'cons', round(d['overhead_vs_ideal_consistent_median'],3), 'pre', d['preempt_random_median'])"
timeout 1200 python scripts/live_c3_c4.py --seeds 2 --repeats 1 --iterations 20 --workloads $W --variants priority --tag scan64 --out gpurun_out/m19_live_s64_p$pass > gpurun_out/m19_live_s64_p$pass.log 2>&1; echo "scan64 rc=$?"
grep SUMMARY gpurun_out/m19_live_s64_p$pass.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l[8:]); print('  s64', d['workload'], 'cons', round(d['ms_consistent_median'],2), 'rand', round(d['ms_random_median'],2), 'vs ideal rand', round(d['overhead_vs_ideal_random_median'],3), 'cons', round(d['overhead_vs_ideal_consistent_median'],3), 'pre', d['preempt_random_median'])"
done
timeout 900 python -m pytest tests/test_gpu_sched.py tests/test_gpu_live.py tests/test_gpu_subcomm.py -q --timeout 600 -p no:cacheprovider > gpurun_out/m19_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/m19_tests.log
