#!/bin/bash
# profiling tool: stepping-kernel CTA size (RINSHAN_BLOCK) x table multicast (RINSHAN_CLUSTER) at small batches
for rep in 1 2; do
for cfg in "0 1" "128 1" "64 1" "64 2" "64 4" "128 2"; do
  set -- $cfg
  echo "== block $1 cluster $2"
  RINSHAN_BLOCK=$1 RINSHAN_CLUSTER=$2 python bench.py --sweep 2048,4096,8192,16384 --no-cpu-baseline --no-e2e --steps 60 --warmup 5 2>/dev/null | grep sweep | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('  n=%d  %.1f us  %.1f M' % (d['envs'], d['ms_per_launch']*1e3, d['env_steps_per_s']/1e6))"
done; done
