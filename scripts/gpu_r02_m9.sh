#!/bin/bash
cd "$GRAFT_REPO_ROOT"
W=c3,resnet50-buckets,resnet50-tensors,bert-large-buckets
for pass in 1 2; do
OCCL_LIB_PATH=paper_2303_06324_b200/lib/exp/lib_m8.so timeout 1200 python scripts/live_c3_c4.py --seeds 3 --repeats 1 --iterations 20 --workloads $W --variants priority --tag m8 --out gpurun_out/m9_live_m8_p$pass > gpurun_out/m9_live_m8_p$pass.log 2>&1; echo "m8 rc=$?"; grep SUMMARY gpurun_out/m9_live_m8_p$pass.log | cut -c1-260
timeout 1200 python scripts/live_c3_c4.py --seeds 3 --repeats 1 --iterations 20 --workloads $W --variants priority --tag nonfront --out gpurun_out/m9_live_nf_p$pass > gpurun_out/m9_live_nf_p$pass.log 2>&1; echo "nf rc=$?"; grep SUMMARY gpurun_out/m9_live_nf_p$pass.log | cut -c1-260
done
timeout 600 python scripts/stickiness_case.py --out gpurun_out/m9_stickiness_case > gpurun_out/m9_stickiness.log 2>&1; echo "stickiness rc=$?"; cut -c1-250 gpurun_out/m9_stickiness.log | tail -4
