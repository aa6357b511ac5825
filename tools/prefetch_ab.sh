#!/bin/bash
# profiling tool: L1 prefetch of the env lines (RINSHAN_PREFETCH 0/1/2): bench value + sweeps fresh/steady
for rep in 1 2; do
for p in ${PREFETCH_MODES:-0 1 2}; do
  echo "== prefetch $p"
  RINSHAN_PREFETCH=$p python bench.py --steps 200 --warmup 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('  bench value %.1f M e2e %.1f M fused %.1f M' % (d['value']/1e6, d['e2e']['value']/1e6, d['fused_rollout']['value']/1e6))"
  RINSHAN_PREFETCH=$p python bench.py --sweep 4096,16384,65536,1048576 --no-cpu-baseline --no-e2e --steps 50 --warmup 5 2>/dev/null | grep sweep | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('  fresh n=%d  %.1f us  %.1f M' % (d['envs'], d['ms_per_launch']*1e3, d['env_steps_per_s']/1e6))"
  RINSHAN_PREFETCH=$p python bench.py --sweep 4096,1048576 --sweep-warm 200 --no-cpu-baseline --no-e2e --steps 50 --warmup 5 2>/dev/null | grep sweep | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('  steady n=%d  %.1f us  %.1f M' % (d['envs'], d['ms_per_launch']*1e3, d['env_steps_per_s']/1e6))"
done; done
