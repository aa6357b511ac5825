#!/bin/bash
# profiling tool: envs per warp at the bench batch with lane groups (bench value, fresh + steady rollout)
for e in 1 2 4 8; do
  echo "== RINSHAN_EPW=$e"
  RINSHAN_EPW=$e python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-e2e --no-fused 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  try: d=json.loads(l)
  except Exception: continue
  print('  bench value %.1f M' % (d['value']/1e6))
"
  RINSHAN_EPW=$e python tools/kstep_large.py 4096 2>&1
done
