# dev: A/B token plans overlapping the batch kernel (DP_DEV_PLAN_OVERLAP=1) vs queued behind it
for r in 1 2 3; do for c in ${CFGS:-cfg4r cfg4b cfg4}; do for o in 0 1; do
  printf "%s overlap=%s " $c $o; DP_DEV_PLAN_OVERLAP=$o python bench.py --config $c --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']/1e6,1), d['roofline']['frac'], d['e2e']['value'])"
done; done; done
