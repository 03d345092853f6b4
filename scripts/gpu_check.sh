#!/bin/bash
# GPU check after a change: selected -m gpu test files (args, default: the fast set) + a bench line.
cd "$GRAFT_REPO_ROOT"
TESTS="${TESTS:-tests/test_gpu_hazards.py tests/test_gpu_subcomm.py tests/test_gpu_sched.py tests/test_gpu_live.py tests/test_gpu_parity.py}"
TAG="${TAG:-check}"
timeout 2400 python -m pytest $TESTS -v --timeout 600 -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/${TAG}_tests.log
if [ -z "$NOBENCH" ]; then
timeout 600 python bench.py --steps 20 --warmup 5 ${BENCH_ARGS:-} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
cut -c1-400 gpurun_out/${TAG}_bench.json
fi
