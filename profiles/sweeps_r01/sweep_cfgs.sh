# bench parameter sweep; configs one per line in file $1
mkdir -p gpurun_out
while read -r cfg; do
  [ -z "$cfg" ] && continue
  echo "== $cfg"
  timeout 300 python bench.py --no-e2e --no-cpu --steps 10 --warmup 3 $cfg 2>&1 | python -c "import json,sys
for l in sys.stdin:
  try: d=json.loads(l)
  except Exception: print(l.strip()[:300]); continue
  p=d['probes']
  print('busbw', round(d['value'],1), 'ms', round(d['ms_per_step'],3), 'frac', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'], 'run/commit', p['per_commit_cycles']['cycRun'], 'poll', p['per_commit_cycles']['cycPoll'], 'data', p['per_slice_data_cycles'], 'dwait', p['per_slice_datawait_cycles'])"
done < "$1"
