python -m pytest tests/test_gpu_parity.py tests/test_scenarios.py tests/test_gpu_golden.py -m gpu -q -x > gpurun_out/r2an_tests.log 2>&1
for rep in 1 2; do for v in chi ring; do RINSHAN_LIB=build_variants/$v.so python bench.py --steps 150 --warmup 5 --no-cpu-baseline --no-e2e --row-steps 10 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v', 'value %.1f' % (d['value']/1e6), 'med %.1f us' % (d['launch_ms']['median']*1e3), 'fused %.1f' % (d['fused_rollout']['value']/1e6), ' '.join('%s/%d %.1f' % (r['rule'], r['envs_per_gpu'], r['value']/1e6) for r in d['rows']))
" >> gpurun_out/r2an_ab.txt; done; done
