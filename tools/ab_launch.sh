#!/bin/bash
# A/B: warm ncu launch-list times of kernels matching $1 for each ab/lib*.so
cd "$(dirname "$0")/.."
for lib in ab/lib*.so; do
  n=$(basename "$lib" .so)
  KST_LIB_PATH=$PWD/$lib ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
    --log-file gpurun_out/ab_$n.csv python tools/one_frame.py 2001 2 > /dev/null 2>&1
  echo "== $n $(python tools/launches.py gpurun_out/ab_$n.csv 0.5 2>/dev/null | grep -E "$1" | tr -s ' ' | tr '\n' ';')"
done
