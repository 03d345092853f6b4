# quick loop: GPU tests + bench (+ optional extra command in $1)
set -x
mkdir -p gpurun_out
if [ -z "$SKIP_TESTS" ]; then timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/gputest.log; fi
timeout 600 python bench.py --check --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
if [ -n "$1" ]; then eval "$1"; fi
