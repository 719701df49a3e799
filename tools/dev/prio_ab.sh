# dev: plan stream at the highest priority (default) vs the lowest (DP_DEV_PLAN_PRIO=0)
for r in 1 2 3; do for c in ${CFGS:-cfg4 cfg4r cfg4b cfg2 cfg5}; do for o in 1 0; do
  printf "%s prio=%s " $c $o; DP_DEV_PLAN_PRIO=$o python bench.py --config $c --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']/1e6,1), d['roofline']['frac'], round(d['e2e']['value']/1e6,3) if d.get('e2e') else None)"
done; done; done
