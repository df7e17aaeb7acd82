#!/bin/bash
# one GPU iteration: the GPU test suite, the pose-kernel timing diagnostic and
# a short bench with per-kernel timings
python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python tools/diag_pose.py 2>&1 | tail -9 | head -4
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-batch 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value']); [print(k, round(v['avg_us'],2), round(v['us_per_frame'],1)) for k,v in d['kernels'].items()]"
