#!/bin/bash
# live-arrival threshold sweep (priority / FIFO): which spin base / cap / stall gate keep random orders near consistent
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hazards.py -x -q --timeout 300 -p no:cacheprovider > gpurun_out/r02c_parity.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/r02c_parity.log
W=c3,resnet50-buckets,bert-large-buckets
COMMON="--seeds 2 --repeats 1 --iterations 10 --fifo-iterations 3 --fifo-seeds 2 --workloads $W"
i=0
for knobs in "--spin-cap 65536" "--spin-cap 8192" "--spin-cap 4096" "--spin-base 1024 --spin-step 128 --spin-min 64 --spin-cap 2048" \
             "--spin-base 512 --spin-step 64 --spin-min 32 --spin-cap 1024" "--spin-cap 8192 --stall-ns 50000" ; do
  i=$((i+1))
  timeout 900 python scripts/live_c3_c4.py $COMMON $knobs --tag "k$i: $knobs" --out gpurun_out/r02c_live_k$i > gpurun_out/r02c_live_k$i.log 2>&1; echo "k$i rc=$?"
  grep SUMMARY gpurun_out/r02c_live_k$i.log | cut -c1-330
done
