#!/bin/bash
# Round-2 first GPU call: the new parity cases against the round-1 build, plus a baseline bench line.
cd "$GRAFT_REPO_ROOT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02_smi.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_hazards.py -v --timeout 200 -p no:cacheprovider > gpurun_out/r02_hazards_old_all.log 2>&1 || true
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_old.json 2> gpurun_out/r02_bench_old.err || true
