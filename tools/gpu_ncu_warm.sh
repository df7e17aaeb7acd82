#!/bin/bash
# ncu --set full without cache flushing between replays (warm L2, as inside the
# frame graph). usage: tools/gpu_ncu_warm.sh <kernel-regex> <tag> [skip] [count]
k=$1; tag=$2; skip=${3:-10}; cnt=${4:-2}
mkdir -p gpurun_out/$tag
python tools/profile_frame.py c3 3 > gpurun_out/$tag/plain.log 2>&1 && \
ncu --set full --cache-control none --clock-control none --import-source on -k regex:$k -s $skip -c $cnt -o gpurun_out/$tag/prof python tools/profile_frame.py c3 3 > gpurun_out/$tag/ncu.log 2>&1
tail -1 gpurun_out/$tag/ncu.log
