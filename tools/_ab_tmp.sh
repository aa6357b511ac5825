for rep in 1 2; do for v in cand kind3; do
RINSHAN_LIB=build_variants/$v.so python bench.py --sweep 131072,262144,1048576 --steps 30 --warmup 3 --sweep-warm 200 2>/dev/null | python -c "
import sys,json
print('$v sweep', ' '.join('%d:%.1f' % (d['envs'], d['env_steps_per_s']/1e6) for d in map(json.loads, sys.stdin)))" >> gpurun_out/r2x_ab.txt
RINSHAN_LIB=build_variants/$v.so RINSHAN_ORDER=2 python bench.py --sweep 16384,65536 --steps 60 --warmup 3 --sweep-warm 200 2>/dev/null | python -c "
import sys,json
print('$v order2', ' '.join('%d:%.1f' % (d['envs'], d['env_steps_per_s']/1e6) for d in map(json.loads, sys.stdin)))" >> gpurun_out/r2x_ab.txt
done; done
