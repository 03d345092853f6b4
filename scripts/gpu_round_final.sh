# tests + multiprocess + sanitizer + ncu launch list + ncu full capture of the daemon + bench (+reference)
bash scripts/gpu_check_all.sh
bash scripts/gpu_sanitize.sh
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:occl_daemon -c 1 -o gpurun_out/prof_daemon -f python bench.py --steps 2 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
timeout -s KILL 600 python bench.py --check > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"; cat gpurun_out/bench_final.json
timeout -s KILL 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref.json
