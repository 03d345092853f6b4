#!/bin/bash
# Round-2 final pass B: live C3/C4 at 10 seeds x 3 repeats (priority) and 3 x 3 (FIFO variants), C3 back to
# back, latency vs size for every kind, the C2 sweep at 8 virtual ranks.
cd "$GRAFT_REPO_ROOT"
timeout 3000 python scripts/live_c3_c4.py --seeds 10 --repeats 3 --iterations 200 --fifo-iterations 10 --fifo-seeds 3 --out gpurun_out/fb_live > gpurun_out/fb_live.log 2>&1; echo "live rc=$?"
timeout 900 python scripts/live_c3_c4.py --seeds 10 --repeats 3 --fifo-seeds 3 --workloads c3 --c3-gap zero --tag b2b --out gpurun_out/fb_live_b2b > gpurun_out/fb_live_b2b.log 2>&1; echo "live b2b rc=$?"
for f in gpurun_out/fb_live.log gpurun_out/fb_live_b2b.log; do grep SUMMARY $f | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l[8:]); print(d['tag'], d['workload'], d['variant'], d['runs'], 'cons', round(d['ms_consistent_median'],2), 'rand', round(d['ms_random_median'],2), 'ovh', round(d['overhead_median'],3), 'vs ideal rand', round(d['overhead_vs_ideal_random_median'],3), 'cons', round(d['overhead_vs_ideal_consistent_median'],3), 'pre', d['preempt_random_median'])"; done
timeout 1200 python scripts/latency_split.py --tag final --out gpurun_out/fb_lat > gpurun_out/fb_lat.log 2>&1; echo "lat rc=$?"
timeout 1500 python scripts/sweep_c2.py --out gpurun_out/fb_c2_sweep > gpurun_out/fb_c2.log 2>&1; echo "c2 rc=$?"; tail -3 gpurun_out/fb_c2.log | cut -c1-200
