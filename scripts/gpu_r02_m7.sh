#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python scripts/trace_live.py --runs 30 --policy 1 --out gpurun_out/m7_trace_live_p1.json > gpurun_out/m7_trace_live_p1.log 2>&1; echo "p1 rc=$?"; grep -c makespan gpurun_out/m7_trace_live_p1.log; tail -1 gpurun_out/m7_trace_live_p1.log
