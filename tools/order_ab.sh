#!/bin/bash
# profiling tool: env ordering on / off at large batches, fresh and steady state
for o in 1 0; do
  echo "== RINSHAN_ORDER=$o"
  RINSHAN_ORDER=$o python bench.py --sweep 131072,262144,1048576 --no-cpu-baseline --no-e2e --steps 50 --warmup 5 2>&1 | grep sweep | cut -c1-140
  RINSHAN_ORDER=$o python tools/kstep_large.py 2>&1
done
