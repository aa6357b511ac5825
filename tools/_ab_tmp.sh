for rep in 1 2; do for pf in 1 2; do RINSHAN_PREFETCH=$pf python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --no-fused --row-steps 20 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('pf$pf', 'value %.1f' % (d['value']/1e6), 'med %.1f us' % (d['launch_ms']['median']*1e3), ' '.join('%s/%d %.1f' % (r['rule'], r['envs_per_gpu'], r['value']/1e6) for r in d['rows']))
" >> gpurun_out/r2ax_ab.txt
RINSHAN_PREFETCH=$pf python bench.py --sweep 16384,65536,262144 --steps 40 --warmup 3 --sweep-warm 200 2>/dev/null | python -c "
import sys,json
print('   pf$pf sweep', ' '.join('%d:%.1f' % (d['envs'], d['env_steps_per_s']/1e6) for d in map(json.loads, sys.stdin)))" >> gpurun_out/r2ax_ab.txt
done; done
