set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sched.py -x -q -p no:cacheprovider > gpurun_out/gputest_q.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gputest_q.log
bash scripts/sweep_cfgs.sh ${SWEEPFILE:-scripts/sweep2.txt}
