# per-lane tempty arrive (OCCL_LANE_ARRIVE=1 build in lib/exp) vs the elected-lane arrive
mkdir -p gpurun_out
L=paper_2303_06324_b200/lib/exp/libocclb200_lane.so
for i in 1 2 3; do
  echo "== default"; timeout -s KILL 300 python bench.py --no-e2e --no-cpu --steps 10 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['roofline']['frac'],3))"
  echo "== lane"; OCCL_LIB_PATH=$L timeout -s KILL 300 python bench.py --no-e2e --no-cpu --steps 10 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['roofline']['frac'],3))"
done
OCCL_LIB_PATH=$L timeout -s KILL 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/lane_pt.log 2>&1; echo "lane pytest rc=$?"; tail -1 gpurun_out/lane_pt.log
OCCL_LIB_PATH=$L timeout -s KILL 900 compute-sanitizer --tool racecheck --print-limit 100000 python scripts/sanitize_small.py > gpurun_out/san_racecheck_lane.log 2>&1; echo "racecheck rc=$?"; tail -2 gpurun_out/san_racecheck_lane.log
