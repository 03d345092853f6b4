set -x

timeout 1500 python scripts/mixed_c3.py --seeds 1 --workloads c3,resnet50-tensors,resnet50-buckets,bert-large-buckets --variants priority:1,priority:0,fifo:1 --out gpurun_out/c3_c4 > gpurun_out/c3.log 2>&1; echo "c3 rc=$?"
python -c "
import json
for l in open('gpurun_out/c3_c4.jsonl'):
    d=json.loads(l); print(d['workload'], d['order_policy'], d['stickiness'], round(d['ms_consistent'],2), round(d['ms_random'],2), round(d['preemption_overhead'],3), d['consistent']['preemptions'], d['random']['preemptions'])
"
