#!/bin/bash
# profiling tool: shared-memory stage (RINSHAN_STAGE=1) vs default on the final build
for rep in 1 2; do
for st in 0 1; do
  echo "== RINSHAN_STAGE=$st"
  RINSHAN_STAGE=$st python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-fused 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('  bench value %.1f M e2e %.1f M launch median %.1f us' % (d['value']/1e6, d['e2e']['value']/1e6, d['launch_ms']['median']*1e3))"
  RINSHAN_STAGE=$st python bench.py --sweep 1024,16384 --no-cpu-baseline --no-e2e --steps 100 --warmup 5 2>/dev/null | grep sweep | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('  n=%d  %.1f us  %.1f M' % (d['envs'], d['ms_per_launch']*1e3, d['env_steps_per_s']/1e6))"
done; done
