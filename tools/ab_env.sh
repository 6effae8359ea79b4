#!/bin/bash
# A/B of environment switches: pipeline time (tools/quick_bench.py) and the ncu launch-list
# times of kernels matching $1, for each setting in $AB_ENVS (space-separated, "-" = none)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in ${AB_ENVS:--}; do
  e=${v/-/}
  echo "== ${v}"
  env $e python tools/quick_bench.py 2001 2>&1 | grep -E "pipeline|lrkron" | tail -3
  if [ -n "$1" ]; then
    env $e ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/ab_env.csv python tools/one_frame.py 2001 3 > /dev/null 2>&1
    python tools/launches.py gpurun_out/ab_env.csv 0.33 2>/dev/null | grep -E "$1"
  fi
done
