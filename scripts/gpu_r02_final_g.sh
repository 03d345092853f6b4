#!/bin/bash
# Round-2 final pass G (the final source): the whole -m gpu suite, smoke, bench line, ncu launch list + full
# capture, both 10,000-trial campaigns, live C3/C4 (priority, 10 seeds x 3), C3 back to back, straggler case,
# latency split vs size for every kind, C2 pipelined sweep.
cd "$GRAFT_REPO_ROOT"
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/fg_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/fg_tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fg_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/fg_smoke.log | cut -c1-200
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/fg_bench.json 2> gpurun_out/fg_bench.err; echo "bench rc=$?"; cut -c1-300 gpurun_out/fg_bench.json
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/fg_bench2.json 2> gpurun_out/fg_bench2.err; echo "bench2 rc=$?"; cut -c1-200 gpurun_out/fg_bench2.json
bash scripts/gpu_ncu.sh
timeout 1500 python scripts/latency_split.py --out gpurun_out/fg_latency_split > gpurun_out/fg_latency.log 2>&1; echo "latency rc=$?"
timeout 1800 python scripts/campaign.py --mode live --trials 10000 --seed0 200000 --out gpurun_out/fg_campaign_live > gpurun_out/fg_campaign_live.log 2>&1; echo "campaign live rc=$?"; tail -1 gpurun_out/fg_campaign_live.log | cut -c1-300
timeout 2400 python scripts/campaign.py --mode fifo --trials 10000 --seed0 300000 --out gpurun_out/fg_campaign_fifo > gpurun_out/fg_campaign_fifo.log 2>&1; echo "campaign fifo rc=$?"; tail -1 gpurun_out/fg_campaign_fifo.log | cut -c1-300
timeout 2400 python scripts/live_c3_c4.py --seeds 10 --repeats 3 --iterations 200 --variants priority --out gpurun_out/fg_live > gpurun_out/fg_live.log 2>&1; echo "live rc=$?"
timeout 900 python scripts/live_c3_c4.py --seeds 10 --repeats 3 --workloads c3 --c3-gap zero --variants priority --tag b2b --out gpurun_out/fg_live_b2b > gpurun_out/fg_live_b2b.log 2>&1; echo "live b2b rc=$?"
for f in gpurun_out/fg_live.log gpurun_out/fg_live_b2b.log; do grep SUMMARY $f | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l[8:]); print(d['tag'], d['workload'], d['variant'], d['runs'], 'cons', round(d['ms_consistent_median'],2), 'rand', round(d['ms_random_median'],2), 'ovh', round(d['overhead_median'],3), 'vs ideal rand', round(d['overhead_vs_ideal_random_median'],3), 'cons', round(d['overhead_vs_ideal_consistent_median'],3), 'pre', d['preempt_random_median'])"; done
timeout 600 python scripts/stickiness_case.py --out gpurun_out/fg_stickiness_case > gpurun_out/fg_stickiness.log 2>&1; echo "stickiness rc=$?"; cut -c1-200 gpurun_out/fg_stickiness.log | tail -4
timeout 1200 python scripts/sweep_c2.py --out gpurun_out/fg_c2_sweep > gpurun_out/fg_c2.log 2>&1; echo "c2 rc=$?"
