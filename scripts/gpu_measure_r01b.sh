# measurement refresh: C2 sweep, C3/C4 mixes
set -x
mkdir -p gpurun_out
timeout 1800 python scripts/sweep_c2.py --out gpurun_out/c2_sweep > gpurun_out/c2.log 2>&1; echo "c2 rc=$?"; cat gpurun_out/c2_sweep.md
timeout 2400 python scripts/mixed_c3.py --seeds 2 --variants priority:1,priority:0,fifo:1,fifo:0 --out gpurun_out/c3_c4 > gpurun_out/c3.log 2>&1; echo "c3 rc=$?"
python -c "
import json
for l in open('gpurun_out/c3_c4.jsonl'):
    d=json.loads(l); print(d['workload'], d['order_policy'], d['stickiness'], d['seed'], round(d['ms_consistent'],2), round(d['ms_random'],2), round(d['preemption_overhead'],3), d['consistent']['preemptions'], d['random']['preemptions'])
"
