RINSHAN_LIB=build_variants/_rinshan_sloc.so timeout 600 python -m pytest tests/test_gpu_soak.py -x -q -k "lane_group or ordering" > gpurun_out/sloc.log 2>&1
for rep in 1 2; do for v in b0 sloc; do
  echo "== $v"
  RINSHAN_LIB=build_variants/_rinshan_$v.so python bench.py --sweep 4096,16384,65536,262144,1048576 --no-cpu-baseline --no-e2e --steps 40 --warmup 5 2>/dev/null | grep sweep | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('  n=%d  %.1f us  %.1f M' % (d['envs'], d['ms_per_launch']*1e3, d['env_steps_per_s']/1e6))"
  RINSHAN_LIB=build_variants/_rinshan_$v.so python bench.py --sweep 1048576 --sweep-warm 150 --no-cpu-baseline --no-e2e --steps 20 --warmup 3 2>/dev/null | grep sweep | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('  steady n=%d  %.1f us  %.1f M' % (d['envs'], d['ms_per_launch']*1e3, d['env_steps_per_s']/1e6))"
done; done >> gpurun_out/sloc.log 2>&1
