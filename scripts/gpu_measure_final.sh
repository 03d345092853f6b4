# end-of-round measurement: tests, C2 sweep, C3/C4, C5, latency, stickiness case, ncu, bench (+reference)
set -x
mkdir -p gpurun_out
timeout -s KILL 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout -s KILL 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -s --timeout 300 > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|campaign" gpurun_out/gputest.log | tail -4
timeout -s KILL 1500 python scripts/sweep_c2.py --out gpurun_out/c2_sweep > gpurun_out/c2.log 2>&1; echo "c2 rc=$?"
timeout -s KILL 1800 python scripts/mixed_c3.py --seeds 2 --variants priority:1,priority:0,fifo:1,fifo:0 --out gpurun_out/c3_c4 > gpurun_out/c3.log 2>&1; echo "c3 rc=$?"
timeout -s KILL 600 python scripts/hybrid_c5.py --out gpurun_out/c5_hybrid > gpurun_out/c5.log 2>&1; echo "c5 rc=$?"
timeout -s KILL 300 python scripts/latency_single.py > gpurun_out/latency_single.jsonl 2>&1; echo "lat rc=$?"
for cfg in "--spin-base 4096 --spin-cap 65536" "--spin-base 1024 --spin-cap 8192" "--spin-base 256 --spin-cap 2048"; do timeout -s KILL 300 python scripts/stickiness_case.py $cfg --out gpurun_out/sc_$(echo $cfg | tr -d " -") > /dev/null 2>&1; done; cat gpurun_out/sc_*.jsonl > gpurun_out/stickiness_case_all.jsonl
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:occl_daemon -c 1 -o gpurun_out/prof_daemon -f python bench.py --steps 2 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
timeout -s KILL 600 python bench.py --check > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout -s KILL 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2>&1; echo "ref rc=$?"
