#!/bin/bash
# profiling tool: shared-memory carveout preference (RINSHAN_CARVEOUT, percent of the max) at small and large batches
for rep in 1 2; do
for c in default 0 25 40 60 100; do
  echo "== carveout $c"
  if [ $c = default ]; then unset RINSHAN_CARVEOUT; else export RINSHAN_CARVEOUT=$c; fi
  python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-e2e --no-fused 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('  bench value %.1f M launch median %.1f us' % (d['value']/1e6, d['launch_ms']['median']*1e3))"
  python bench.py --sweep 16384,65536,1048576 --no-cpu-baseline --no-e2e --steps 30 --warmup 5 2>/dev/null | grep sweep | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('  n=%d  %.1f us  %.1f M' % (d['envs'], d['ms_per_launch']*1e3, d['env_steps_per_s']/1e6))"
done; done
