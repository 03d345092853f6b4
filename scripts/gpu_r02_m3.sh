#!/bin/bash
# Round-2 pass 3: LL speculation (parity + latency), bandwidth variants (L2 prefetch, chunking), FIFO diagnosis.
cd "$GRAFT_REPO_ROOT"
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sched.py -q --timeout 600 -p no:cacheprovider > gpurun_out/m3_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/m3_tests.log
for spec in 0 1; do for b in 4096 65536; do
  timeout 300 python scripts/trace_ll.py --bytes $b --ll-spec $spec --out gpurun_out/m3_trace_ll_s${spec}_$b.json 2>&1 | tail -1
done; done
timeout 900 python scripts/latency_split.py --kinds allreduce --ll-spec 1 --tag llspec --out gpurun_out/m3_lat_llspec > gpurun_out/m3_lat_llspec.log 2>&1; echo "lat llspec rc=$?"
bash scripts/gpu_variants.sh scripts/var_r02c.txt vc 2 0
timeout 120 python scripts/probe_multicast.py > gpurun_out/m3_multicast.json 2>&1; echo "probe rc=$?"; tail -c 1500 gpurun_out/m3_multicast.json
timeout 900 python scripts/fifo_diagnosis.py --seeds 1 --out gpurun_out/m3_fifo_diag.jsonl > gpurun_out/m3_fifo_diag.log 2>&1; echo "fifo diag rc=$?"; cut -c1-500 gpurun_out/m3_fifo_diag.log | tail -4
