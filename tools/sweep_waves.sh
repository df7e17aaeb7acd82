python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for e in "WT_WAVE_SHAPE=1" "WT_WAVE_SHAPE=44" "WT_WAVE_POSE=2" "WT_WAVE_POSE=4" "WT_WAVE_POSE=8" "WT_WAVE_SEARCH=4" "WT_WAVE_SEARCH=16"; do
  echo "== $e"; env $e python tools/batch_timing.py 64 2>&1 | grep -E "B=|shape_step|pose_system|search|normals|stats"
done
python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C3', round(d['value']), round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value'])); [print('  ', k, round(v['avg_us'],2), round(v['us_per_frame'],1)) for k,v in d['kernels'].items()]"
