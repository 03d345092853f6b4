#!/bin/bash
# DRAM traffic per bench variant (ncu single-pass metrics on one daemon launch of 4 steps) + interleaved timing.
cd "$GRAFT_REPO_ROOT"
VARIANTS=("--l2-hints 2" "--l2-hints 3" "--l2-hints 2 --conn-slots 4" "--l2-hints 3 --conn-slots 4" "--l2-hints 3 --slice-kib 160" "--l2-hints 3 --slice-kib 128 --conn-slots 6")
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct
i=0
for v in "${VARIANTS[@]}"; do
  i=$((i+1))
  timeout 600 ncu --metrics $M --clock-control none -k regex:occl_daemon -c 1 --csv python bench.py --steps 4 --warmup 0 --no-e2e --no-cpu --no-conn-only $v > gpurun_out/traffic_v$i.csv 2> gpurun_out/traffic_v$i.err
  echo "v$i [$v] rc=$?"; grep -E "dram__bytes|gpu__time|lts__t_bytes|hit_rate" gpurun_out/traffic_v$i.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
for pass in 1 2; do
  i=0
  for v in "${VARIANTS[@]}"; do
    i=$((i+1))
    timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu --no-conn-only $v > gpurun_out/traffic_bench_v${i}_p$pass.json 2>/dev/null
    echo "pass $pass v$i [$v] $(python -c "import json;d=json.loads(open('gpurun_out/traffic_bench_v${i}_p$pass.json').readline());print(round(d['value'],1), round(d['roofline']['frac'],3))")"
  done
done
