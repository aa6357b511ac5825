#!/bin/bash
# profiling tool: bench.py value / e2e for build variants, alternating
for rep in 1 2 3; do
for v in "$@"; do
  RINSHAN_LIB=build_variants/$v.so python bench.py --steps 200 --warmup 10 --no-cpu-baseline 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  try: d=json.loads(l)
  except Exception: continue
  print('$v', 'value %.1f M' % (d['value']/1e6), 'e2e %.1f M' % (d['e2e']['value']/1e6), 'launch median %.1f us' % (d['launch_ms']['median']*1000))
"
done
done
