timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for c in 3 4 5b; do timeout 600 python bench.py --config $c --no-cpu --steps 3 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']; print('cfg', d['config']['workload'][:8], d['value'], d['ms_per_step'], round(r['achieved'],2), round(r['frac'],3))"; done
