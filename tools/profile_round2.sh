#!/bin/bash
# One GPU call of evidence for profiles/: both bench lines (C3 headline, C5
# batch), the ncu launch list of the C3 bench command, and `--set full`
# captures of every kernel of one C3 frame and one C5 batch frame
# (summarised on the box by tools/profile_batch.sh).
# Usage (under gpurun): tools/profile_round2.sh <tag>
set -u
tag=${1:-r01}
out=gpurun_out/$tag
mkdir -p $out
python bench.py --steps 30 --warmup 5 > $out/bench_c3.json 2> $out/bench_c3.err || exit 1
python bench.py --config c5 --steps 10 --warmup 3 > $out/bench_c5.json 2> $out/bench_c5.err || exit 2
cmd="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-batch"
$cmd > $out/plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_c3.csv $cmd \
  > $out/ncu_launches.log 2>&1
bash tools/profile_batch.sh $tag both
