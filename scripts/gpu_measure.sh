# measurement round: tests (incl. 10k-trial campaign), bench, C2 sweep, C3/C4
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider -s > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|campaign" gpurun_out/gputest.log | tail -5
timeout 600 python bench.py --check > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json
timeout 1800 python scripts/sweep_c2.py --out gpurun_out/c2_sweep > gpurun_out/c2.log 2>&1; echo "c2 rc=$?"; cat gpurun_out/c2_sweep.md
timeout 2400 python scripts/mixed_c3.py --out gpurun_out/c3_c4 > gpurun_out/c3.log 2>&1; echo "c3 rc=$?"; tail -30 gpurun_out/c3.log | cut -c1-400
