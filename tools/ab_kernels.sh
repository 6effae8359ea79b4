#!/bin/bash
# A/B kernel timings: for each ab/lib*.so, an ncu launch list of 6 frames (last 3 averaged).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for lib in ab/lib*.so; do
  n=$(basename "$lib" .so)
  KST_LIB_PATH=$PWD/$lib ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/ab_$n.csv python tools/one_frame.py 2001 6 > /dev/null 2>&1
  echo "== $n"; python tools/launches.py gpurun_out/ab_$n.csv | grep -E "${1:-.}" | head -${2:-12}
done
