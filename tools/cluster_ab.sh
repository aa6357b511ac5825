#!/bin/bash
# profiling tool: table-multicast cluster size A/B (RINSHAN_CLUSTER) — bench value, K=1 sweep, fused sweep
for c in 1 2 4 1 2 4; do
  echo "== cluster $c"
  RINSHAN_CLUSTER=$c python bench.py --steps 200 --warmup 20 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('bench value %.1f M e2e %.1f M fused %.1f M' % (d['value']/1e6, d['e2e']['value']/1e6, d.get('fused_rollout',{}).get('value',0)/1e6))"
  RINSHAN_CLUSTER=$c python bench.py --sweep 4096,16384,65536,1048576 --no-cpu-baseline --no-e2e --steps 50 --warmup 5 2>/dev/null | grep sweep | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('  n=%d  %.1f us  %.1f M' % (d['envs'], d['ms_per_launch']*1e3, d['env_steps_per_s']/1e6))"
done
