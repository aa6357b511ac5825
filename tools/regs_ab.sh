for rep in 1 2; do
for v in b0 m6 m7 m8; do for e in 1 2; do
  r=$(RINSHAN_LIB=build_variants/_rinshan_$v.so RINSHAN_EPW=$e python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('value %.1f M launch median %.1f us fused %.1f M' % (d['value']/1e6, d['launch_ms']['median']*1e3, (d.get('fused_rollout') or {}).get('value',0)/1e6))")
  echo "$v epw=$e $r"
done; done; done
