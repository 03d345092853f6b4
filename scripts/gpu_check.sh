# full GPU test suite + bench + scheduler trace
set -x
mkdir -p gpurun_out
timeout -s KILL 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout -s KILL 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -s --durations=8 > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|campaign|FAILED|Error" gpurun_out/gputest.log | tail -12
timeout -s KILL 600 python scripts/trace_sched.py 2>&1 | tail -2
timeout -s KILL 600 python bench.py --no-cpu --check > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print('busbw', round(d['value'],1), 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],2), d['check'], d['clocks'])"
