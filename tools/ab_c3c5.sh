#!/bin/bash
# per-variant (with tools/ab.sh): parity subset, C5 batch frame time (x3), C3 bench (x3)
python -m pytest tests/test_gpu_parity_bench.py tests/test_gpu_golden.py tests/test_gpu_batch.py tests/test_kats.py -m gpu -q -x -k "not c4" 2>&1 | tail -1
python tools/batch_timing.py 64 2>&1 | grep -vE "^\s*$"
for r in 2 3; do python tools/batch_timing.py 64 2>&1 | grep -E "B="; done
for r in 1 2 3; do
python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-batch 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']; print('C3', round(d['value']), round(d['ms_per_step'],4), ' '.join(f'{n}={v[\"avg_us\"]:.1f}' for n,v in k.items()))"
done
