mkdir -p gpurun_out
for n in 8 4 2; do
  timeout -s KILL 1200 python scripts/sweep_c2.py --ranks $n --out gpurun_out/c2_sweep_n$n > gpurun_out/c2_n$n.log 2>&1; echo "c2 n=$n rc=$?"
done
ls gpurun_out
