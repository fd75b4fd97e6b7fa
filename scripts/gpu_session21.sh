export SB_SYNC_TIMEOUT_S=600 PYTHONUNBUFFERED=1
for a in "c2 dense 12" "c2 interval 12" "c2 interval 14" "c3 interval 12" "c3 interval 14"; do
  timeout 900 python -u scripts/exact_bench.py $a > gpurun_out/exact_$(echo $a | tr ' ' _).json 2>/dev/null; echo "$a rc=$?"; cat gpurun_out/exact_$(echo $a | tr ' ' _).json
done
