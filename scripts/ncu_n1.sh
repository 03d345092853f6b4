set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:occl_daemon -c 1 -o gpurun_out/prof_n1 -f python bench.py --steps 2 --warmup 0 --no-e2e --no-cpu --ranks 1 > gpurun_out/ncu_n1.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_n1.log
