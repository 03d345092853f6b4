#!/bin/bash
# Round-2 re-entry: the whole -m gpu suite, the smoke, one bench line and the ncu launch list + full capture.
cd "$GRAFT_REPO_ROOT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/v_smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/v_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/v_tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/v_bench.json 2> gpurun_out/v_bench.err; echo "bench rc=$?"; cut -c1-600 gpurun_out/v_bench.json
python -c "
import json;d=json.loads(open('gpurun_out/v_bench.json').readline())
print({k:d.get(k) for k in ('value','ms_per_step','gpu_launches','clocks')}); print(d.get('roofline')); print(d.get('e2e')); print({k:v for k,v in d.items() if k not in ('roofline','e2e','config','clocks','cpu_baseline')})"
bash scripts/gpu_ncu.sh
