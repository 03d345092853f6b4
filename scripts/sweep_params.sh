# bench parameter sweep (no e2e / cpu legs); configs from $SWEEP (one per line) or defaults
mkdir -p gpurun_out
CFGS="${SWEEP:-
--grid-blocks 18
--grid-blocks 16
--grid-blocks 18 --pipe-depth 4
--grid-blocks 18 --slice-kib 128 --conn-slots 4
--grid-blocks 18 --slice-kib 32 --conn-slots 8 --slices-per-chunk 4
--grid-blocks 18 --conn-slots 8 --slices-per-chunk 4
--grid-blocks 18 --threads 320}"
echo "$CFGS" | while read -r cfg; do
  [ -z "$cfg" ] && continue
  echo "== $cfg"
  timeout 300 python bench.py --no-e2e --no-cpu $cfg 2>&1 | python -c "import json,sys
for l in sys.stdin:
  try: d=json.loads(l)
  except Exception: print(l.strip()[:300]); continue
  print('busbw', round(d['value'],1), 'ms', round(d['ms_per_step'],3), 'frac', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons']); print('  probes', d.get('probes'))"
done
