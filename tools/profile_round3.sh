#!/bin/bash
# Round-2 evidence in one GPU call (under gpurun): the default bench line,
# the ncu launch list of the bench command, `--set full` captures of every
# kernel of one C3 frame, one C5 batch frame and one C4 frame (summarised on
# the box), and traffic.json from them.
# Usage: tools/profile_round3.sh <tag>
set -u
tag=${1:-r02}
out=gpurun_out/$tag
mkdir -p $out /tmp/ncu_$tag
python bench.py > $out/bench_default.json 2> $out/bench_default.err || exit 1
cmd="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-batch"
$cmd > $out/plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches_c3.csv $cmd \
  > $out/ncu_launches.log 2>&1
bash tools/profile_batch.sh $tag both > $out/profile_batch.log 2>&1
K='regex:"k_(fk|ingest|skin|normals|pixoff|scatter|search|pose_system|pose_solve|shape|shape_after)(<|\$)"'
python tools/profile_frame.py c4 3 > $out/plain_c4.log 2>&1 &&
eval ncu --set full --clock-control none -k $K -s 55 -c 55 -o /tmp/ncu_$tag/c4_frame -f \
  python tools/profile_frame.py c4 3 > $out/ncu_c4.log 2>&1
python tools/ncu_summary.py /tmp/ncu_$tag/c4_frame.ncu-rep > $out/ncu_c4_frame.md
python tools/traffic_json.py c3=$out/ncu_c3_frame.md c5=$out/ncu_batch_frame.md c4=$out/ncu_c4_frame.md > $out/traffic.json
ls -la $out
