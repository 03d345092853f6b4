# compute-sanitizer over a small end-to-end run of the daemon
mkdir -p gpurun_out
timeout -s KILL 120 python scripts/sanitize_small.py > gpurun_out/san_plain.log 2>&1; echo "plain rc=$?"; tail -2 gpurun_out/san_plain.log
for tool in memcheck synccheck racecheck; do
  timeout -s KILL 900 compute-sanitizer --tool $tool --print-limit 100000 python scripts/sanitize_small.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/san_$tool.log
done
