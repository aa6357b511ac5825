#!/bin/bash
# profiling tool: A/B build variants (sweep + steady-state k_step / rollout)
for rep in 1 2; do
for spec in "$@"; do
  v=${spec%%:*}; envs=""; [[ "$spec" == *:* ]] && envs=${spec#*:}
  echo "== $spec rep $rep"
  env $envs RINSHAN_LIB=build_variants/$v.so python bench.py --sweep 4096,16384,65536,262144,1048576 --no-cpu-baseline --no-e2e --steps 50 --warmup 5 2>&1 | python -c "
import sys,json
out=[]
for l in sys.stdin:
  try: d=json.loads(l)
  except Exception: continue
  if d.get('sweep'): out.append('%d:%.1f' % (d['envs'], d['env_steps_per_s']/1e6))
print('  sweep M/s', ' '.join(out))
"
  env $envs RINSHAN_LIB=build_variants/$v.so python tools/kstep.py 4096 2>&1 | tail -2
done
done
