#!/bin/bash
cd "$GRAFT_REPO_ROOT"
bash scripts/gpu_variants.sh scripts/var_r02e.txt ve 2 0
timeout 1500 python scripts/sweep_c2.py --out gpurun_out/m17_c2_sweep > gpurun_out/m17_c2.log 2>&1; echo "c2 rc=$?"; grep allreduce gpurun_out/m17_c2_sweep.md
timeout 1200 python scripts/latency_split.py --kinds allreduce,allgather --tag final2 --out gpurun_out/m17_lat > gpurun_out/m17_lat.log 2>&1; echo "lat rc=$?"
python -c "
import json
for l in open('gpurun_out/m17_lat.jsonl'):
    d=json.loads(l); s=d['split'] or {}
    print(d['kind'][:6], d['bytes'], 'e2e med', round(d['e2e_median_us'],1), {k:(round(v,2) if isinstance(v,float) else v) for k,v in s.items()})"
