#!/bin/bash
# profiling tool: env ordering forced on / off at mid-size batches, fresh and steady state
for o in 2 0; do
  echo "== RINSHAN_ORDER=$o"
  RINSHAN_ORDER=$o python bench.py --sweep 16384,32768,65536,131072 --no-cpu-baseline --no-e2e --steps 50 --warmup 5 2>&1 | grep sweep | cut -c1-140
  RINSHAN_ORDER=$o python tools/kstep_large.py 16384,32768,65536,131072 2>&1
done
