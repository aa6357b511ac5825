#!/bin/bash
# profiling tool: out-of-line engine members (build variants) - bench-size sweep, alternating
for rep in 1 2; do for v in ${VARIANTS:-b0}; do
  RINSHAN_LIB=build_variants/_rinshan_$v.so python bench.py --sweep 1024,4096,16384,262144 --no-cpu-baseline --no-e2e --steps 100 --warmup 5 2>/dev/null | grep sweep | python -c "
import json,sys
r=[]
for l in sys.stdin:
    d=json.loads(l); r.append('%d:%.1fM' % (d['envs'], d['env_steps_per_s']/1e6))
print('$v', ' '.join(r))"
  RINSHAN_LIB=build_variants/_rinshan_$v.so python bench.py --sweep 4096 --fuse 100 --no-cpu-baseline --no-e2e --steps 3 --warmup 1 2>/dev/null | grep sweep | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v fused100 %.1f M' % (d['env_steps_per_s']/1e6))"
done; done
