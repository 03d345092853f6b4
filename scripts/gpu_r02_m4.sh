#!/bin/bash
# Round-2 pass 4: TMA SQ fetch + rate-limited host polls: full GPU suite, latency split, LL trace,
# a short live C3/C4 check of the priority policy, bench line.
cd "$GRAFT_REPO_ROOT"
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/m4_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/m4_tests.log
timeout 900 python scripts/latency_split.py --kinds allreduce --tag tmasq --out gpurun_out/m4_lat > gpurun_out/m4_lat.log 2>&1; echo "lat rc=$?"
python -c "
import json
for l in open('gpurun_out/m4_lat.jsonl'):
    d=json.loads(l); s=d['split'] or {}
    print(d['kind'][:6], d['bytes'], 'e2e med', round(d['e2e_median_us'],1), {k:(round(v,2) if isinstance(v,float) else v) for k,v in s.items()})"
timeout 300 python scripts/trace_ll.py --bytes 4096 --out gpurun_out/m4_trace_ll.json 2>&1 | tail -1
timeout 1200 python scripts/live_c3_c4.py --seeds 2 --repeats 1 --iterations 20 --fifo-iterations 3 --fifo-seeds 1 --workloads c3,resnet50-buckets,bert-large-buckets --variants priority,fifo+stickiness --out gpurun_out/m4_live > gpurun_out/m4_live.log 2>&1; echo "live rc=$?"; grep SUMMARY gpurun_out/m4_live.log | cut -c1-330
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/m4_bench.json 2> gpurun_out/m4_bench.err; echo "bench rc=$?"; cut -c1-200 gpurun_out/m4_bench.json
