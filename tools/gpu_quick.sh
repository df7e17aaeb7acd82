#!/bin/bash
# quick GPU iteration: parity suite, C5 batch timing, C3 bench summary
python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python tools/batch_timing.py 64 2>&1 | tail -12
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-batch 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C3', round(d['value']), round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value'])); [print('  ', k, round(v['avg_us'],2), round(v['us_per_frame'],1)) for k,v in d['kernels'].items()]"
