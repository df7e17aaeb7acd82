#!/bin/bash
# A/B timing of prebuilt library variants in _alt/*.so (experiments only):
#   tools/ab.sh "<command>"   -- runs <command> once per variant
cp paper_1711_07999_b200/libwt_gpu.so /tmp/ab_cur.so
for so in _alt/*.so; do
  cp "$so" paper_1711_07999_b200/libwt_gpu.so
  echo "== $so"
  bash -c "$1"
done
cp /tmp/ab_cur.so paper_1711_07999_b200/libwt_gpu.so
