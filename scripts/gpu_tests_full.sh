set -x
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -s --durations=15 > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|campaign|FAILED|Error" gpurun_out/gputest.log | tail -15; tail -22 gpurun_out/gputest.log
