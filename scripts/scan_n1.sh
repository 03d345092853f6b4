for cfg in "--pipe-depth 2" "--pipe-depth 8" "--pipe-depth 8 --slice-kib 256 --conn-slots 3" "--pipe-depth 8 --slice-kib 1024 --conn-slots 3" "--pipe-depth 4 --slice-kib 256 --conn-slots 3"; do
  timeout 300 python bench.py --no-e2e --no-cpu --ranks 1 $cfg 2>&1 | python -c "import json,sys
for l in sys.stdin:
  try: d=json.loads(l)
  except Exception: print(l.strip()[:200]); continue
  S=d['config']['size_bytes_per_rank']; t=d['ms_per_step']/1e3
  print('n1 $cfg', 'ms',round(d['ms_per_step'],3),'traffic TB/s',round(2*S/t/1e12,2),'per-SM GB/s',round(2*S/t/1e9/18,1), d['probes']['per_slice_data_cycles'], d['probes']['per_slice_datawait_cycles'])"
done
for cfg in "--pipe-depth 8" "--pipe-depth 8 --slice-kib 128 --conn-slots 4" "--pipe-depth 8 --conn-slots 8 --slices-per-chunk 4"; do
  timeout 300 python bench.py --no-e2e --no-cpu $cfg 2>&1 | python -c "import json,sys
for l in sys.stdin:
  try: d=json.loads(l)
  except Exception: print(l.strip()[:200]); continue
  print('n8 $cfg', 'busbw', round(d['value'],1), 'ms',round(d['ms_per_step'],3), d['probes'])"
done
