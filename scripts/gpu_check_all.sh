bash scripts/gpu_check.sh
timeout -s KILL 900 python -m pytest tests/test_gpu_multiprocess.py -q -p no:cacheprovider > gpurun_out/mp.log 2>&1; echo "mp rc=$?"; tail -2 gpurun_out/mp.log
