# round-end style GPU check: tests, smoke, bench lines (logs under gpurun_out/)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider ${PYTEST_ARGS:-} > gpurun_out/gputest2.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/gputest2.log | grep -E "FAILED|passed|failed"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke2.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke2.log
if [ -z "$NOBENCH" ]; then
timeout 300 python bench.py > gpurun_out/bench2.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench2.log
timeout 300 python bench.py --config lmode --no-cpu-baseline > gpurun_out/bench2_lmode.log 2>&1; echo "lmode rc=$?"; tail -1 gpurun_out/bench2_lmode.log
fi
