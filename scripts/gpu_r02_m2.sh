#!/bin/bash
# Round-2 measurement pass 2: host-read microbenchmark, the two 10,000-trial campaigns,
# live C3/C4 (10 seeds x 3 repeats), the stickiness case study.
cd "$GRAFT_REPO_ROOT"
timeout 60 ./scripts/micro/hostread > gpurun_out/m2_hostread.json 2>&1; echo "hostread rc=$?"; cat gpurun_out/m2_hostread.json
timeout 1500 python scripts/campaign.py --mode fifo --trials 10000 --out gpurun_out/m2_campaign > gpurun_out/m2_campaign_fifo.log 2>&1; echo "campaign fifo rc=$?"; tail -2 gpurun_out/m2_campaign_fifo.log
timeout 1800 python scripts/campaign.py --mode live --trials 10000 --seed0 100000 --out gpurun_out/m2_campaign > gpurun_out/m2_campaign_live.log 2>&1; echo "campaign live rc=$?"; tail -2 gpurun_out/m2_campaign_live.log
timeout 2400 python scripts/live_c3_c4.py --seeds 10 --repeats 3 --iterations 200 --fifo-iterations 10 --fifo-seeds 3 --out gpurun_out/m2_live > gpurun_out/m2_live.log 2>&1; echo "live rc=$?"; grep SUMMARY gpurun_out/m2_live.log | cut -c1-400
timeout 600 python scripts/stickiness_case.py --out gpurun_out/m2_stickiness_case > gpurun_out/m2_stickiness.log 2>&1; echo "stickiness rc=$?"; tail -4 gpurun_out/m2_stickiness.log | cut -c1-400
