set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --deselect tests/test_gpu_campaign.py::test_deadlock_campaign_8_ranks > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed" gpurun_out/gputest.log | tail -3
timeout 1500 python scripts/mixed_c3.py --seeds 1 --workloads c3,resnet50-tensors --out gpurun_out/c3_c4 > gpurun_out/c3.log 2>&1; echo "c3 rc=$?"; cut -c1-330 gpurun_out/c3.log | tail -12
timeout 1800 python scripts/sweep_c2.py --out gpurun_out/c2_sweep > gpurun_out/c2.log 2>&1; echo "c2 rc=$?"; cat gpurun_out/c2_sweep.md; tail -3 gpurun_out/c2.log
