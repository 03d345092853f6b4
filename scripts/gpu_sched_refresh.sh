mkdir -p gpurun_out
timeout -s KILL 1500 python scripts/mixed_c3.py --seeds 2 --variants priority:1 --out gpurun_out/c3_c4_prio > gpurun_out/c3p.log 2>&1; echo "c3 rc=$?"; tail -12 gpurun_out/c3p.log
timeout -s KILL 600 python scripts/hybrid_c5.py --seeds 2 --policies 1 --out gpurun_out/c5_prio > gpurun_out/c5p.log 2>&1; echo "c5 rc=$?"; tail -6 gpurun_out/c5p.log
