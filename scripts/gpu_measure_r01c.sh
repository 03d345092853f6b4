# measurement refresh after LL / SQ mirror: C2 sweep, C3/C4, C5, single-op latency, bench sweep
set -x
mkdir -p gpurun_out
timeout -s KILL 1500 python scripts/sweep_c2.py --out gpurun_out/c2_sweep > gpurun_out/c2.log 2>&1; echo "c2 rc=$?"; cat gpurun_out/c2_sweep.md
timeout -s KILL 1800 python scripts/mixed_c3.py --seeds 2 --variants priority:1,priority:0,fifo:1,fifo:0 --out gpurun_out/c3_c4 > gpurun_out/c3.log 2>&1; echo "c3 rc=$?"
timeout -s KILL 600 python scripts/hybrid_c5.py --out gpurun_out/c5_hybrid > gpurun_out/c5.log 2>&1; echo "c5 rc=$?"
timeout -s KILL 300 python scripts/latency_single.py > gpurun_out/latency_single.jsonl 2>&1; echo "lat rc=$?"
cat > /tmp/sw.txt <<'EOT'
--grid-blocks 18 --slice-kib 256 --conn-slots 4
--grid-blocks 18 --slice-kib 256 --conn-slots 3
--grid-blocks 16 --slice-kib 128 --conn-slots 4
--grid-blocks 18 --slice-kib 128 --conn-slots 4 --stages 4
--grid-blocks 18 --slice-kib 192 --conn-slots 4
EOT
timeout -s KILL 400 bash scripts/sweep_cfgs.sh /tmp/sw.txt
