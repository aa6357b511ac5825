#!/bin/bash
for e in 1 2 4 8 32; do
  echo "== epw $e"
  RINSHAN_EPW=$e python tools/cycles.py 4096 2>&1
  RINSHAN_EPW=$e python bench.py --sweep 4096,16384 --no-cpu-baseline --no-e2e --steps 50 --warmup 5 2>&1 | grep sweep | cut -c1-140
done
