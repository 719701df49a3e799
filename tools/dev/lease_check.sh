# dev: group-lease change -- full GPU suite, GetNext host cost, host-bound configs
python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
bash tools/dev/gn_prof.sh 2>&1 | head -1
for c in cfg1 cfg4 cfg4r cfg4b cfg2; do printf "%s " $c; python bench.py --config $c --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['e2e']['value'] if d.get('e2e') else None)"; done
