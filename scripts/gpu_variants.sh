#!/bin/bash
# Interleaved bench variants: bash scripts/gpu_variants.sh <variants.txt> <tag> [passes] [traffic]
# one variant (bench.py flags) per line; every pass runs each variant once; with traffic=1 each
# variant also gets one ncu single-pass capture of DRAM / L2 bytes on a 4-step daemon launch.
cd "$GRAFT_REPO_ROOT"
VF="$1"; TAG="$2"; PASSES="${3:-2}"; TRAFFIC="${4:-0}"
mapfile -t VARIANTS < "$VF"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct
for pass in $(seq 1 $PASSES); do
  i=0
  for v in "${VARIANTS[@]}"; do
    i=$((i+1))
    # a line "LIB=<path> flags..." runs that variant against another build of the library
    unset OCCL_LIB_PATH
    if [[ "$v" == LIB=* ]]; then export OCCL_LIB_PATH="${v%% *}"; OCCL_LIB_PATH="${OCCL_LIB_PATH#LIB=}"; v="${v#* }"; [[ "$v" == LIB=* ]] && v=""; fi
    timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu --no-conn-only $v > gpurun_out/${TAG}_v${i}_p$pass.json 2> gpurun_out/${TAG}_v${i}_p$pass.err
    echo "pass $pass v$i [$v] $(python -c "import json;d=json.loads(open('gpurun_out/${TAG}_v${i}_p$pass.json').readline());print(round(d['value'],1), round(d['roofline']['frac'],3), d['probes']['cycles_per_release_fence'], d['probes']['per_slice_data_cycles'], d['probes']['per_commit_cycles']['cycRun'])" 2>&1 | tail -1)"
  done
done
if [ "$TRAFFIC" = "1" ]; then
  i=0
  for v in "${VARIANTS[@]}"; do
    i=$((i+1))
    unset OCCL_LIB_PATH
    if [[ "$v" == LIB=* ]]; then export OCCL_LIB_PATH="${v%% *}"; OCCL_LIB_PATH="${OCCL_LIB_PATH#LIB=}"; v="${v#* }"; [[ "$v" == LIB=* ]] && v=""; fi
    timeout 600 ncu --metrics $M --clock-control none -k regex:occl_daemon -c 1 --csv python bench.py --steps 4 --warmup 0 --no-e2e --no-cpu --no-conn-only $v > gpurun_out/${TAG}_traffic_v$i.csv 2> gpurun_out/${TAG}_traffic_v$i.err
    echo "traffic v$i [$v] rc=$?"; grep -E "dram__bytes|gpu__time|lts__t_bytes|hit_rate" gpurun_out/${TAG}_traffic_v$i.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
  done
fi
