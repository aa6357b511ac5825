#!/bin/bash
# profiling tool: register caps at large batches (fresh + steady sweeps) per build variant
for rep in 1 2; do
for v in b0 r3 r5; do
  echo "== $v"
  RINSHAN_LIB=build_variants/_rinshan_$v.so python bench.py --sweep 262144,1048576 --no-cpu-baseline --no-e2e --steps 20 --warmup 3 2>/dev/null | grep sweep | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('  fresh n=%d  %.1f us  %.1f M' % (d['envs'], d['ms_per_launch']*1e3, d['env_steps_per_s']/1e6))"
  RINSHAN_LIB=build_variants/_rinshan_$v.so python bench.py --sweep 1048576 --sweep-warm 150 --no-cpu-baseline --no-e2e --steps 20 --warmup 3 2>/dev/null | grep sweep | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('  steady n=%d  %.1f us  %.1f M' % (d['envs'], d['ms_per_launch']*1e3, d['env_steps_per_s']/1e6))"
done; done
