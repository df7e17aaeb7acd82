#!/bin/bash
# per-variant: GPU tests + C3 bench summary (used with tools/ab.sh)
python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for r in 1 2; do
python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-batch 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C3', round(d['value']), round(d['ms_per_step'],4), 'search', round(d['kernels']['search+average']['avg_us'],2))"
done
