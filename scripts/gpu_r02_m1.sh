#!/bin/bash
# Round-2 measurement pass 1 on the regression-fixed build: full -m gpu suite, bench line,
# latency split vs size (three CQ variants), NVLS probe, FIFO thrash diagnosis, ncu.
cd "$GRAFT_REPO_ROOT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/m1_smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/m1_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/m1_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/m1_bench.json 2> gpurun_out/m1_bench.err; echo "bench rc=$?"; cut -c1-300 gpurun_out/m1_bench.json
timeout 120 python scripts/probe_multicast.py > gpurun_out/m1_multicast.json 2>&1; echo "probe rc=$?"; tail -2 gpurun_out/m1_multicast.json
for cq in 0 1 2; do
  timeout 900 python scripts/latency_split.py --kinds allreduce --cq-mode $cq --tag cq$cq --out gpurun_out/m1_lat_cq$cq > gpurun_out/m1_lat_cq$cq.log 2>&1; echo "lat cq$cq rc=$?"
done
timeout 900 python scripts/latency_split.py --kinds allgather,reducescatter,broadcast --sizes 4096,65536,262144,1048576,16777216 --tag kinds --out gpurun_out/m1_lat_kinds > gpurun_out/m1_lat_kinds.log 2>&1; echo "lat kinds rc=$?"
timeout 1500 python scripts/fifo_diagnosis.py --seeds 2 --out gpurun_out/m1_fifo_diag.jsonl > gpurun_out/m1_fifo_diag.log 2>&1; echo "fifo diag rc=$?"; tail -8 gpurun_out/m1_fifo_diag.log | cut -c1-400
bash scripts/gpu_ncu.sh
