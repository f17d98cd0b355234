set -e
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for c in 2 4; do timeout 300 python bench.py --config $c --no-cpu --steps 10 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']; print('cfg', d['config']['workload'][:8], d['value'], d['ms_per_step'], r['kernel'][:40], round(r['achieved'],2), round(r['frac'],3), d['e2e']['value'])"; done
