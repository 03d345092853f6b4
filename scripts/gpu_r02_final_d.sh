#!/bin/bash
# Round-2 final pass D: C5 hybrid sub-communicators (pre-enqueued, both policies), C2 sweeps at 2 and 4 virtual ranks.
cd "$GRAFT_REPO_ROOT"
timeout 1200 python scripts/hybrid_c5.py --out gpurun_out/fd_c5 > gpurun_out/fd_c5.log 2>&1; echo "c5 rc=$?"; tail -6 gpurun_out/fd_c5.log | cut -c1-300
for r in 2 4; do
  timeout 1200 python scripts/sweep_c2.py --ranks $r --kinds allreduce,allgather,reducescatter --out gpurun_out/fd_c2_n$r > gpurun_out/fd_c2_n$r.log 2>&1; echo "c2 n$r rc=$?"; grep -E "allreduce \| (4096|1048576|268435456|1073741824) " gpurun_out/fd_c2_n$r.md
done
timeout 300 python scripts/trace_ll.py --bytes 4096 --out gpurun_out/fd_trace_ll.json 2>&1 | tail -1 | cut -c1-3000
