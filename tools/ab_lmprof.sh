#!/bin/bash
# A/B of L-mode window phase profiles (libs built with -DKST_LM_PROF) + the sweep parity tests
cd "$(dirname "$0")/.."
for lib in ab/lib*.so; do
  n=$(basename "$lib" .so)
  echo "== $n"
  KST_LIB_PATH=$PWD/$lib python tools/lm_prof.py 256 81 | grep -E "rounds hist|eig|total"
  KST_LIB_PATH=$PWD/$lib python tools/lm_prof.py 2001 81 | grep -E "rounds hist|eig|total"
  KST_LIB_PATH=$PWD/$lib timeout 600 python -m pytest -q -p no:cacheprovider tests/test_gpu_lmode_batched.py 2>&1 | tail -1
done
