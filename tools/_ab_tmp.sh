for rep in 1 2; do for st in 0 1; do RINSHAN_STAGE=$st python bench.py --steps 150 --warmup 5 --no-cpu-baseline --row-steps 10 --no-rows 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('stage $st', 'value %.1f' % (d['value']/1e6), 'med %.1f us' % (d['launch_ms']['median']*1e3), 'e2e %.1f' % (d['e2e']['value']/1e6), 'fused %.1f' % (d['fused_rollout']['value']/1e6))
" >> gpurun_out/r2ak_ab.txt; done; done
