python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python tools/diag_pose.py 2>&1 | tail -9
python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value']); [print(k, round(v['avg_us'],2), round(v['us_per_frame'],1)) for k,v in d['kernels'].items()]"
mkdir -p gpurun_out/pose
python tools/profile_frame.py c3 3 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_pose -s 10 -c 2 -o gpurun_out/pose/pose python tools/profile_frame.py c3 3 > gpurun_out/pose/ncu.log 2>&1; tail -1 gpurun_out/pose/ncu.log
