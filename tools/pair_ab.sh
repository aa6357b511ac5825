#!/bin/bash
# profiling tool: CTA-tile pairing by step kind on / off at small batches, fresh and steady state
for p in 1 0; do
  echo "== RINSHAN_PAIR=$p"
  RINSHAN_PAIR=$p python bench.py --sweep 4096,16384,65536 --no-cpu-baseline --no-e2e --steps 50 --warmup 5 2>&1 | grep sweep | cut -c1-140
  RINSHAN_PAIR=$p python tools/kstep_large.py 4096,16384,65536 2>&1
  RINSHAN_PAIR=$p python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-e2e --no-fused 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  try: d=json.loads(l)
  except Exception: continue
  print('  bench value %.1f M' % (d['value']/1e6))
"
done
