# A/B of the p=10 dense union variants (SB_UNION_VARIANT) on C3 + parity per variant
export SB_SYNC_TIMEOUT_S=120 PYTHONUNBUFFERED=1
for v in 5 6 7 8; do
  SB_UNION_VARIANT=$v timeout 300 python -u -m pytest tests -m gpu -x -q -k "golden or c1 or random" > gpurun_out/pytest_v$v.log 2>&1; echo "v$v pytest rc=$?"; tail -1 gpurun_out/pytest_v$v.log
done
for v in 0 5 6 7 8 0; do
  SB_UNION_VARIANT=$v timeout 300 python -u bench.py --no-cpu --no-e2e --no-variants --steps 2 --warmup 1 > gpurun_out/ab_v$v.json 2> gpurun_out/ab_v$v.log; echo "v$v rc=$?"; grep "union avg" gpurun_out/ab_v$v.log
done
