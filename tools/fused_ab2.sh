#!/bin/bash
# profiling tool: default bench.py (200 steps) value / e2e / fused per build variant
for rep in 1 2; do for v in ${VARIANTS:-b0}; do
  RINSHAN_LIB=build_variants/_rinshan_$v.so python bench.py --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); print('$v value %.1f M e2e %.1f M fused %.1f M' % (d['value']/1e6, d['e2e']['value']/1e6, d['fused_rollout']['value']/1e6))"
done; done
