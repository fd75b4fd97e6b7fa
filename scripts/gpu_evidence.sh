#!/usr/bin/env bash
# Regenerates the GPU evidence under gpurun_out/ (copy what you keep to profiles/).
# Run on a B200 box from the repo root, e.g.
#   gpurun --timeout 3600 -- bash scripts/gpu_evidence.sh [tests|bench|ncu|sweeps|widened|all]
# Each step is bounded by its own timeout; nothing here is a bench value when run under ncu.
set -u
export SB_SYNC_TIMEOUT_S=600 PYTHONUNBUFFERED=1
what=${1:-all}
mkdir -p gpurun_out
run() { echo "== $*" >> gpurun_out/evidence.log; "$@"; echo "rc=$? ($1 ${*: -1})" >> gpurun_out/evidence.log; }

if [[ $what == tests || $what == all ]]; then
  run timeout 1500 python -u -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
  run timeout 300 python -u -c "import __graft_entry__ as g; g.smoke()"
fi
if [[ $what == bench || $what == all ]]; then
  run timeout 900 python -u bench.py --local > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.log
  run timeout 600 python -u bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.log
  run timeout 600 python -u scripts/e2e_breakdown.py > gpurun_out/e2e_breakdown.txt 2>&1
  run timeout 600 python -u scripts/e2e_small.py > gpurun_out/e2e_small_graphs.txt 2>&1
  run timeout 600 python -u bench.py --config c2 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.log
  run timeout 600 python -u bench.py --config c1 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.log
  run timeout 600 python -u scripts/step_overhead.py > gpurun_out/step_overhead.json 2>/dev/null
fi
if [[ $what == ncu || $what == all ]]; then
  # launch list of the bench command + one full capture of the dense union kernel
  run timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_c3.csv python -u bench.py --profile --no-cpu --no-e2e --no-variants --no-pipeline
  run timeout 900 ncu --set full --clock-control none --import-source on -k regex:union_kernel -s 3 -c 1 \
      -o gpurun_out/prof_union python -u bench.py --profile --no-cpu --no-e2e --no-variants --no-pipeline
  run timeout 600 ncu --set full --clock-control none --import-source on -k regex:union_interval -s 3 -c 1 \
      -o gpurun_out/prof_interval python -u scripts/pipeline_profile.py c3
  run timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_pipeline.csv python -u scripts/pipeline_profile.py c3
  run timeout 900 ncu --set full --clock-control none --import-source on -k regex:local_kernel -s 1 -c 1 \
      -o gpurun_out/prof_local python -u scripts/profile_local.py 117000 4096
fi
if [[ $what == sweeps || $what == all ]]; then
  run timeout 900 python -u scripts/sweep.py > gpurun_out/sweeps.json 2> gpurun_out/sweeps.log
  run timeout 1500 python -u scripts/shard_projection.py c3 > gpurun_out/shard_projection.json 2>/dev/null
  run timeout 1500 python -u scripts/hilbert_c3.py c3 > gpurun_out/hilbert_c3.json 2>/dev/null
fi
if [[ $what == widened || $what == all ]]; then
  run timeout 900 python -u scripts/accuracy_table.py > gpurun_out/accuracy_table.json 2>/dev/null
  run timeout 1500 python -u scripts/accuracy_scale.py c2 c3 > gpurun_out/accuracy_scale.json 2>/dev/null
  for a in "c2 interval 12" "c3 interval 12"; do
    run timeout 900 python -u scripts/exact_bench.py $a > "gpurun_out/exact_${a// /_}.json" 2>/dev/null
  done
  run timeout 600 python -u scripts/local_metrics_bench.py c3 > gpurun_out/local_c3.json 2>/dev/null
  for tool in memcheck racecheck synccheck; do
    run timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python -u scripts/sanitize_widened.py \
        > gpurun_out/sanitizer_widened_$tool.log 2>&1
  done
fi
