#!/bin/bash
# Round-2 final pass A: the whole -m gpu suite, the smoke, the bench line, ncu launch list + full capture,
# DRAM/L2 traffic of the direct-mode and connector-only variants, compute-sanitizer, both campaigns.
cd "$GRAFT_REPO_ROOT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/fa_smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/fa_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/fa_tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fa_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/fa_smoke.log | cut -c1-200
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/fa_bench.json 2> gpurun_out/fa_bench.err; echo "bench rc=$?"; cut -c1-300 gpurun_out/fa_bench.json
bash scripts/gpu_ncu.sh
printf '%s\n' "" "--force-sys 1" > gpurun_out/fa_var.txt
bash scripts/gpu_variants.sh gpurun_out/fa_var.txt fav 1 1
bash scripts/gpu_sanitize.sh
timeout 1500 python scripts/campaign.py --mode fifo --trials 10000 --out gpurun_out/fa_campaign > gpurun_out/fa_campaign_fifo.log 2>&1; echo "campaign fifo rc=$?"; tail -1 gpurun_out/fa_campaign_fifo.log | cut -c1-300
timeout 1800 python scripts/campaign.py --mode live --trials 10000 --seed0 100000 --out gpurun_out/fa_campaign > gpurun_out/fa_campaign_live.log 2>&1; echo "campaign live rc=$?"; tail -1 gpurun_out/fa_campaign_live.log | cut -c1-300
