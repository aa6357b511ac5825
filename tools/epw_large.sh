#!/bin/bash
# profiling tool: envs-per-warp at large batches (lane groups fill the rest)
for e in 32 16 8; do
  echo "== epw $e"
  RINSHAN_EPW=$e python bench.py --sweep 65536,262144,1048576 --no-cpu-baseline --no-e2e --steps 50 --warmup 5 2>&1 | grep sweep | cut -c1-150
done
