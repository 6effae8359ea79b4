#!/bin/bash
# A/B: for each ab/lib*.so, pipeline time (tools/quick_bench.py, CUDA events) and the
# ncu launch-list times of kernels matching $1
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for lib in ab/lib*.so; do
  n=$(basename "$lib" .so)
  echo "== $n"
  KST_LIB_PATH=$PWD/$lib python tools/quick_bench.py 2001 2>&1 | grep pipeline | tail -2
  if [ -n "$1" ]; then
    KST_LIB_PATH=$PWD/$lib ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/ab_$n.csv python tools/one_frame.py 2001 3 > /dev/null 2>&1
    python tools/launches.py gpurun_out/ab_$n.csv 0.33 | grep -E "$1"
  fi
done
