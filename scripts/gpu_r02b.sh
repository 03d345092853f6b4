#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err; echo "bench rc=$?"
timeout 900 python -m pytest tests/test_gpu_multiprocess.py -v --timeout 600 -p no:cacheprovider > gpurun_out/r02b_mp.log 2>&1; echo "mp rc=$?"; tail -3 gpurun_out/r02b_mp.log
timeout 1500 python scripts/live_c3_c4.py --seeds 2 --repeats 1 --iterations 20 --fifo-iterations 3 --fifo-seeds 1 --out gpurun_out/r02b_live > gpurun_out/r02b_live.log 2>&1; echo "live rc=$?"; grep SUMMARY gpurun_out/r02b_live.log
