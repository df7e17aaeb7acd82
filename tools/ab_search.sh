#!/bin/bash
# per-variant (with tools/ab.sh): parity at the bench configs, C5 batch timing, C3 bench
python -m pytest tests/test_gpu_parity_bench.py tests/test_gpu_golden.py tests/test_gpu_batch.py -m gpu -q -x -k "not c4" 2>&1 | tail -1
python tools/batch_timing.py 64 2>&1 | grep -E "B=|normals|search|skin|pose_sys|shape"
for r in 1 2; do
python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-batch 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']; print('C3', round(d['value']), round(d['ms_per_step'],4), 'search', round(k['search+average']['avg_us'],2), 'normals', round(k['normals+bucket']['avg_us'],2))"
done
