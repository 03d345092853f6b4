#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 600 python scripts/trace_live.py --runs 20 --policy 1 --out gpurun_out/m5_trace_live_p1.json > gpurun_out/m5_trace_live_p1.log 2>&1; echo "p1 rc=$?"; tail -4 gpurun_out/m5_trace_live_p1.log | cut -c1-3000
timeout 600 python scripts/trace_live.py --runs 20 --policy 0 --out gpurun_out/m5_trace_live_p0.json > gpurun_out/m5_trace_live_p0.log 2>&1; echo "p0 rc=$?"; grep makespan gpurun_out/m5_trace_live_p0.log | cut -c1-200 | head -20
timeout 600 python scripts/stickiness_case.py --out gpurun_out/m5_stickiness_case > gpurun_out/m5_stickiness.log 2>&1; echo "stickiness rc=$?"; cut -c1-300 gpurun_out/m5_stickiness.log | tail -4
