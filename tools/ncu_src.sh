#!/bin/bash
# Source-level warp-stall profile of one launch of each named kernel, in the
# C5 batch (tools/batch_timing.py 64) and/or the C3 frame (tools/profile_frame.py):
# ncu --set full --import-source on, then per-line stall tables (tools/ncu_lines.py)
# written next to the raw metrics. Usage (under gpurun):
#   tools/ncu_src.sh <tag> <batch|c3> <kernel> [kernel ...]
set -u
tag=$1; what=$2; shift 2
out=gpurun_out/$tag; mkdir -p $out /tmp/ncs_$tag
if [ "$what" = batch ]; then cmd="python tools/batch_timing.py 64"; skip=20; else cmd="python tools/profile_frame.py c3 3"; skip=12; fi
$cmd > $out/plain_$what.log 2>&1 || exit 1
for k in "$@"; do
  ncu --set full --clock-control none --import-source on -k "regex:^$k(<|\$)" -s $skip -c 1 -o /tmp/ncs_$tag/${what}_$k -f $cmd > $out/ncu_${what}_$k.log 2>&1
  ncu -i /tmp/ncs_$tag/${what}_$k.ncu-rep --page source --csv --print-source cuda,sass > /tmp/ncs_$tag/${what}_$k.csv 2>/dev/null
  python tools/ncu_lines.py /tmp/ncs_$tag/${what}_$k.csv 40 > $out/lines_${what}_$k.txt
  python tools/ncu_summary.py /tmp/ncs_$tag/${what}_$k.ncu-rep > $out/summary_${what}_$k.md
  ncu -i /tmp/ncs_$tag/${what}_$k.ncu-rep --page details --csv > $out/details_${what}_$k.csv 2>/dev/null
done
ls $out
