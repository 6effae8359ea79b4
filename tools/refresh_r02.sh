#!/bin/bash
# r02 final refresh: headline bench line (graph replay), its ncu launch list, L-mode lines, smoke
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python bench.py > gpurun_out/r02_bench.log 2>&1; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r02_launches_gotcha.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
  > gpurun_out/r02_ncu_bench.log 2>&1; echo "ncu rc=$?"
python tools/launches.py gpurun_out/r02_launches_gotcha.csv > gpurun_out/r02_launches_gotcha.txt 2>&1
timeout 300 python bench.py --config lmode --no-cpu-baseline > gpurun_out/r02_bench_lmode.log 2>&1; echo "lmode rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo "smoke rc=$?"
tail -1 gpurun_out/r02_bench.log | cut -c1-300
