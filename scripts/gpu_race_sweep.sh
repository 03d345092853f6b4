mkdir -p gpurun_out
timeout -s KILL 900 compute-sanitizer --tool racecheck --print-limit 100000 python scripts/sanitize_small.py > gpurun_out/san_racecheck3.log 2>&1; echo "racecheck rc=$?"; tail -2 gpurun_out/san_racecheck2.log
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt.log
bash scripts/sweep_cfgs.sh scripts/sweep20.txt
