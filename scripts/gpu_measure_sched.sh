set -x
mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -s --timeout 300 > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|campaign" gpurun_out/gputest.log | tail -4
timeout -s KILL 2400 python scripts/mixed_c3.py --seeds 2 --variants priority:1,priority:0,fifo:1,fifo:0 --out gpurun_out/c3_c4 > gpurun_out/c3.log 2>&1; echo "c3 rc=$?"
timeout -s KILL 600 python scripts/hybrid_c5.py --out gpurun_out/c5_hybrid > gpurun_out/c5.log 2>&1; echo "c5 rc=$?"
for cfg in "--spin-base 4096 --spin-cap 65536" "--spin-base 1024 --spin-cap 8192" "--spin-base 256 --spin-cap 2048"; do timeout -s KILL 300 python scripts/stickiness_case.py $cfg --out gpurun_out/sc_$(echo $cfg | tr -d " -") > /dev/null 2>&1; done; cat gpurun_out/sc_*.jsonl > gpurun_out/stickiness_case_all.jsonl
timeout -s KILL 600 python bench.py --check > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
