export SB_SYNC_TIMEOUT_S=600 PYTHONUNBUFFERED=1
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python -u scripts/sanitize_widened.py > gpurun_out/sanitizer_widened_$tool.log 2>&1; echo "sanitizer $tool rc=$?"; tail -3 gpurun_out/sanitizer_widened_$tool.log
done
SB_LOCAL_GLOBAL=1 timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -u scripts/sanitize_widened.py > gpurun_out/sanitizer_widened_memcheck_global.log 2>&1; echo "memcheck global rc=$?"; tail -2 gpurun_out/sanitizer_widened_memcheck_global.log
timeout 900 python -u scripts/sweep.py > gpurun_out/sweeps.json 2> gpurun_out/sweeps.log; echo sweep rc=$?; grep -v generated gpurun_out/sweeps.log | tail -30
