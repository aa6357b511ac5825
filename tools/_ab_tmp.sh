python -m pytest tests/test_gpu_parity.py tests/test_gpu_soak.py::test_lane_group_sizes_match_oracle tests/test_gpu_soak.py::test_env_ordering_matches_oracle -m gpu -q -x > gpurun_out/r2bd_tests.log 2>&1
for rep in 1 2; do for v in bfree3 bfree2; do RINSHAN_LIB=build_variants/$v.so python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --row-steps 20 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v', 'value %.1f' % (d['value']/1e6), 'med %.1f us' % (d['launch_ms']['median']*1e3), 'fused %.1f' % (d['fused_rollout']['value']/1e6), ' '.join('%s/%d %.1f' % (r['rule'], r['envs_per_gpu'], r['value']/1e6) for r in d['rows']))
" >> gpurun_out/r2bd_ab.txt
RINSHAN_LIB=build_variants/$v.so python bench.py --sweep 16384,65536,262144 --steps 40 --warmup 3 --sweep-warm 200 2>/dev/null | python -c "
import sys,json
print('   $v sweep', ' '.join('%d:%.1f' % (d['envs'], d['env_steps_per_s']/1e6) for d in map(json.loads, sys.stdin)))" >> gpurun_out/r2bd_ab.txt
done; done
