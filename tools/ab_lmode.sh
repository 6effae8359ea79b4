#!/bin/bash
# A/B for the L-mode kernels: for each ab/lib*.so, the Gotcha-scale and 256 L-mode
# launch lists (kernels matching $1)
cd "$(dirname "$0")/.."
for lib in ab/lib*.so; do
  n=$(basename "$lib" .so)
  echo "== $n"
  for q in ${2:-2001 256}; do
    KST_LIB_PATH=$PWD/$lib ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/abl_${n}_$q.csv python tools/one_lmode_frame.py $q 1 > /dev/null 2>&1
    python tools/launches.py gpurun_out/abl_${n}_$q.csv 1.0 | grep -E "$1" | sed "s/^/q=$q /"
  done
done
