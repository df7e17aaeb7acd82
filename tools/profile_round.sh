#!/bin/bash
# One GPU call's worth of evidence for profiles/: the bench line, the ncu
# launch list of the same bench command, and --set full captures of the hot
# kernels on a short tracking run. Usage (under gpurun): tools/profile_round.sh <tag>
set -u
tag=${1:-r01}
out=gpurun_out/$tag
mkdir -p $out
python bench.py --steps 30 --warmup 5 > $out/bench.json 2> $out/bench.err || exit 1
cmd="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-batch"
$cmd > $out/plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv $cmd > $out/ncu_launches.log 2>&1
pcmd="python tools/profile_frame.py c3 3"
$pcmd > $out/plain_prof.log 2>&1 || exit 2
for k in k_search k_pose_system k_pose_solve k_normals k_shape k_scatter k_pixoff k_skin; do
  ncu --set full --clock-control none --import-source on -k regex:"${k}" -s 6 -c 2 -o $out/full_$k $pcmd \
    > $out/ncu_full_$k.log 2>&1
done
# C5 as one batch of 64 sequences: bench line + full captures of its two hottest kernels
python bench.py --config c5 --steps 10 --warmup 3 > $out/bench_c5.json 2> $out/bench_c5.err || exit 3
python tools/batch_timing.py 64 > $out/plain_batch.log 2>&1 || exit 4
for k in k_normals k_search; do
  ncu --set full --clock-control none --import-source on -k regex:"${k}" -s 20 -c 1 -o $out/batch_$k \
    python tools/batch_timing.py 64 > $out/ncu_batch_$k.log 2>&1
done
echo done
