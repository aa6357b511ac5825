#!/bin/bash
# profiling tool: env ordering on/off at mid batches, fresh (100 launches) and steady (after 300 steps)
for rep in 1 2; do
for o in 0 2; do
  echo "== RINSHAN_ORDER=$o"
  RINSHAN_ORDER=$o python bench.py --sweep 65536,131072,262144 --no-cpu-baseline --no-e2e --steps 100 --warmup 5 2>/dev/null | grep sweep | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('  fresh  n=%d  %.1f us  %.1f M' % (d['envs'], d['ms_per_launch']*1e3, d['env_steps_per_s']/1e6))"
  RINSHAN_ORDER=$o python bench.py --sweep 65536,131072,262144 --sweep-warm 300 --no-cpu-baseline --no-e2e --steps 50 --warmup 5 2>/dev/null | grep sweep | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('  steady n=%d  %.1f us  %.1f M' % (d['envs'], d['ms_per_launch']*1e3, d['env_steps_per_s']/1e6))"
done; done
