#!/bin/bash
# ncu evidence for the batched path (C5: 64 C3 sequences in one frame graph)
# and the single-sequence C3 frame: one `--set full` capture of every frame
# kernel of one frame, summarised on the box (the reports themselves are
# too large to bring back). Usage (under gpurun): tools/profile_batch.sh <tag> [batch|c3|both]
set -u
tag=${1:-r01}
what=${2:-both}
out=gpurun_out/$tag
mkdir -p $out /tmp/ncu_$tag
K='regex:"k_(fk|ingest|skin|normals|pixoff|scatter|search|pose_system|pose_solve|shape|shape_after)(<|\$)"'
if [ "$what" != c3 ]; then
  python tools/batch_timing.py 64 > $out/plain_batch.log 2>&1 || exit 1
  # one batch frame = 55 launches (ingest + 54 graph kernels); skip two frames
  eval ncu --set full --clock-control none -k $K -s 110 -c 55 -o /tmp/ncu_$tag/batch_frame -f \
    python tools/batch_timing.py 64 > $out/ncu_batch.log 2>&1
  python tools/ncu_summary.py /tmp/ncu_$tag/batch_frame.ncu-rep > $out/ncu_batch_frame.md
  ncu -i /tmp/ncu_$tag/batch_frame.ncu-rep --page raw --csv > $out/ncu_batch_frame_raw.csv
fi
if [ "$what" != batch ]; then
  python tools/profile_frame.py c3 3 > $out/plain_prof.log 2>&1 || exit 2
  eval ncu --set full --clock-control none -k $K -s 55 -c 55 -o /tmp/ncu_$tag/c3_frame -f \
    python tools/profile_frame.py c3 3 > $out/ncu_c3.log 2>&1
  python tools/ncu_summary.py /tmp/ncu_$tag/c3_frame.ncu-rep > $out/ncu_c3_frame.md
fi
ls -la $out
echo done
