# bench configuration: parity at full size, ncu launch list + full capture, bench + reference arm
set -x
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider --timeout 200 > gpurun_out/fullsize.log 2>&1; echo "fullsize rc=$?"; tail -2 gpurun_out/fullsize.log
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:occl_daemon -c 1 -o gpurun_out/prof_daemon -f python bench.py --steps 2 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
timeout -s KILL 600 python bench.py --check > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json | cut -c1-400
timeout -s KILL 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2>&1; echo "ref rc=$?"
