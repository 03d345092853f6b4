#!/bin/bash
# Latency A/B on one lease: bash scripts/gpu_lat_ab.sh <tag> <passes> <libdir>... (empty libdir = in-tree build)
# per pass and library: 8-rank AR latency split (4 KiB - 1 MiB, 50 reps); then LL hop traces of the in-tree build.
cd "$GRAFT_REPO_ROOT"
TAG="$1"; PASSES="$2"; shift 2
for pass in $(seq 1 $PASSES); do
  i=0
  for lib in "$@"; do
    i=$((i+1))
    if [ "$lib" = "-" ]; then unset OCCL_LIB_PATH; else export OCCL_LIB_PATH="$lib/libocclb200.so"; fi
    timeout 900 python scripts/latency_split.py --kinds allreduce --sizes 4096,65536,262144,1048576 --reps 50 \
      --tag "${TAG}_v${i}" --out gpurun_out/${TAG}_lat_v${i}_p${pass} > gpurun_out/${TAG}_lat_v${i}_p${pass}.log 2>&1
    echo "pass $pass v$i [$lib] rc=$?"; python -c "
import json,sys
for l in open('gpurun_out/${TAG}_lat_v${i}_p${pass}.jsonl'):
    d=json.loads(l); sp=d['split'] or {}
    print(d['bytes'], round(d['e2e_median_us'],1), {k: round(v,1) for k,v in sp.items() if isinstance(v,float)})
" 2>&1 | tail -5
  done
done
unset OCCL_LIB_PATH
for b in 4096 65536; do
  timeout 600 python scripts/trace_ll.py --bytes $b --out gpurun_out/${TAG}_trace_ll_$b.json > gpurun_out/${TAG}_trace_ll_$b.log 2>&1
  echo "trace $b rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/${TAG}_trace_ll_$b.json'))
print({k: d[k] for k in ('detect_us_median','move_us_median','execute_us_median','fetch_to_switchin_us_median')})
print('median', d['hop_parts_us_median']); print('p10', d['hop_parts_us_p10'])"
done
