# memory-traffic rate of the daemon path vs ring size (same per-rank size)
for R in 1 2 4 8; do
  timeout 300 python bench.py --no-e2e --no-cpu --ranks $R $EXTRA 2>&1 | python -c "import json,sys
R=$R
for l in sys.stdin:
  try: d=json.loads(l)
  except Exception: print(l.strip()[:200]); continue
  S=d['config']['size_bytes_per_rank']; t=d['ms_per_step']/1e3
  traffic=R*(2+4*(R-1)/R)*S
  print('ranks',R,'ms',round(d['ms_per_step'],3),'algbw',round(S/t/1e9,1),'busbw',round(d['value'],1),'ring-traffic TB/s',round(traffic/t/1e12,2), 'min-dram TB/s', round(2*R*S/t/1e12,2))"
done
