#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/m12_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/m12_tests.log
timeout 900 python scripts/latency_split.py --tag llspread --out gpurun_out/m12_lat > gpurun_out/m12_lat.log 2>&1; echo "lat rc=$?"
python -c "
import json
for l in open('gpurun_out/m12_lat.jsonl'):
    d=json.loads(l); s=d['split'] or {}
    print(d['kind'][:6], d['bytes'], 'e2e med', round(d['e2e_median_us'],1), {k:(round(v,2) if isinstance(v,float) else v) for k,v in s.items()})"
