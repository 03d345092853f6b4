#!/bin/bash
# Live C3/C4 A/B over library builds: bash scripts/gpu_live_ab.sh <tag> <passes> <name=libpath|current>...
cd "$GRAFT_REPO_ROOT"
TAG="$1"; PASSES="$2"; shift 2
W=c3,resnet50-buckets,resnet50-tensors,bert-large-buckets
for pass in $(seq 1 $PASSES); do
  for spec in "$@"; do
    name="${spec%%=*}"; lib="${spec#*=}"
    unset OCCL_LIB_PATH; [ "$lib" != "current" ] && export OCCL_LIB_PATH="$lib"
    timeout 1200 python scripts/live_c3_c4.py --seeds 2 --repeats 1 --iterations 20 --workloads $W --variants priority --tag "$name" --out gpurun_out/${TAG}_${name}_p$pass > gpurun_out/${TAG}_${name}_p$pass.log 2>&1; echo "$name p$pass rc=$?"
    grep SUMMARY gpurun_out/${TAG}_${name}_p$pass.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l[8:]); print('  ', d['tag'], d['workload'], 'cons', round(d['ms_consistent_median'],2), 'rand', round(d['ms_random_median'],2), 'vs ideal rand', round(d['overhead_vs_ideal_random_median'],3), 'cons', round(d['overhead_vs_ideal_consistent_median'],3), 'pre', d['preempt_random_median'])"
  done
done
