#!/bin/bash
# profiling tool: front-end optimisation level (-Xcicc -O2 vs default -O3) sweep A/B
for rep in 1 2; do for v in ${VARIANTS:-b0 cc2}; do
  echo "== $v"
  RINSHAN_LIB=build_variants/_rinshan_$v.so python bench.py --sweep 1024,4096,16384,65536,262144,1048576 --no-cpu-baseline --no-e2e --steps 100 --warmup 5 2>/dev/null | grep sweep | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('  n=%d  %.1f us  %.1f M' % (d['envs'], d['ms_per_launch']*1e3, d['env_steps_per_s']/1e6))"
  RINSHAN_LIB=build_variants/_rinshan_$v.so python bench.py --sweep 4096 --fuse 100 --no-cpu-baseline --no-e2e --steps 3 --warmup 1 2>/dev/null | grep sweep | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('  fused100 n=%d  %.1f M' % (d['envs'], d['env_steps_per_s']/1e6))"
done; done
