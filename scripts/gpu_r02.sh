#!/usr/bin/env bash
# Round-2 evidence on one B200 (outputs under gpurun_out/; copy what is kept to profiles/r02/):
#   gpurun --timeout 3000 -- bash scripts/gpu_r02.sh [tests|bench|ncu|ncu_sweep|dist|all]...
# Each step has its own timeout; no number printed under ncu is a bench value.
set -u
export SB_SYNC_TIMEOUT_S=600 PYTHONUNBUFFERED=1
mkdir -p gpurun_out
run() { echo "== $*" >> gpurun_out/r02.log; "$@"; echo "rc=$? ($1 ${*: -1})" >> gpurun_out/r02.log; }
(nproc; lscpu | grep 'Model name'; nvidia-smi -L) > gpurun_out/host.txt 2>&1
NCU="ncu --set full --clock-control none --import-source on"
# keep gpurun_out small (it must stay under 64 MiB to come back): text exports + summary, no .ncu-rep
export_rep() {  # $1 = summary key, $2 = report basename (without .ncu-rep)
  [[ -f gpurun_out/$2.ncu-rep ]] || return
  ncu -i gpurun_out/$2.ncu-rep --page details > gpurun_out/$2_details.txt 2>&1
  python -u scripts/ncu_summary.py --out gpurun_out/ncu_summary.json $1 gpurun_out/$2.ncu-rep > /dev/null
  python -u scripts/ncu_lines.py gpurun_out/$2.ncu-rep > gpurun_out/$2_lines.txt 2>&1
  rm -f gpurun_out/$2.ncu-rep
}
for what in "${@:-all}"; do
if [[ $what == parity ]]; then
  run timeout 1800 python -u -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_parity.log 2>&1; tail -3 gpurun_out/pytest_parity.log
fi
if [[ $what == quick ]]; then
  run timeout 600 python -u bench.py --no-cpu --no-variants --no-pipeline --no-e2e > gpurun_out/bench_c3_quick.json 2> gpurun_out/bench_c3_quick.log
fi
if [[ $what == tests || $what == all ]]; then
  run timeout 2400 python -u -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
  run timeout 300 python -u -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
fi
if [[ $what == bench || $what == all ]]; then
  run timeout 900 python -u bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.log
  run timeout 600 python -u bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.log
  run timeout 600 python -u bench.py --config c2 --no-cpu > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.log
  run timeout 600 python -u bench.py --config c1 --no-cpu > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.log
fi
if [[ $what == ncu || $what == all ]]; then
  run timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_c3.csv python -u bench.py --profile --no-cpu --no-e2e --no-variants --no-pipeline
  run timeout 900 $NCU -k regex:union_kernel -s 3 -c 1 -o gpurun_out/prof_c3_p10 \
      python -u bench.py --profile --no-cpu --no-e2e --no-variants --no-pipeline
  export_rep c3_p10 prof_c3_p10
fi
if [[ $what == ncu_sweep || $what == all ]]; then
  for cfg in "c1 10" "c2 10" "c2 4" "c2 6" "c2 14"; do
    set -- $cfg
    run timeout 600 $NCU -k regex:union_kernel -s 2 -c 1 -o gpurun_out/prof_$1_p$2 \
        python -u bench.py --config $1 --p $2 --profile --no-cpu --no-e2e --no-variants --no-pipeline
    export_rep $1_p$2 prof_$1_p$2
  done
  run timeout 600 $NCU -k regex:union_interval -s 3 -c 1 -o gpurun_out/prof_c3_interval \
      python -u scripts/pipeline_profile.py c3
  export_rep c3_p10_interval prof_c3_interval
fi
if [[ $what == dist || $what == all ]]; then
  # the sharded bench path (2 ranks sharing the one GPU: fused P2P + gloo barrier) vs N=1
  run timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
      --master-port 29533 bench.py --gpus 2 --config c3 --steps 3 --warmup 3 --no-cpu --no-variants --no-pipeline \
      > gpurun_out/bench_c3_w2_shared.json 2> gpurun_out/bench_c3_w2_shared.log
fi
if [[ $what == stats ]]; then
  for c in "c3 10" "c2 10"; do
    SB_LIBRARY=paper_2604_08374_b200/libsieveball_cuda_stats.so timeout 600 python -u scripts/group_stats.py $c \
        >> gpurun_out/group_stats.txt 2>&1
  done
fi
if [[ $what == async ]]; then
  run timeout 900 python -u -m pytest tests/test_gpu_async_upload.py -q -x > gpurun_out/pytest_async.log 2>&1; tail -2 gpurun_out/pytest_async.log
fi
if [[ $what == setup ]]; then
  # setup kernels (validation/work items at upload, run index) and the interval end to end
  run timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_pipeline.csv python -u scripts/pipeline_profile.py c3
  run timeout 600 python -u scripts/e2e_breakdown.py > gpurun_out/e2e_breakdown.txt 2>&1
fi
if [[ $what == sweeps || $what == all ]]; then
  run timeout 900 python -u scripts/sweep.py > gpurun_out/sweeps.json 2> gpurun_out/sweeps.log
fi
done
for what in "$@"; do
if [[ $what == ncusass ]]; then
  # per-SASS-instruction executed counts and stall samples of the C3 union (kept as csv)
  run timeout 900 $NCU -k regex:union_kernel -s 3 -c 1 -o gpurun_out/prof_sass \
      python -u bench.py --profile --no-cpu --no-e2e --no-variants --no-pipeline
  ncu -i gpurun_out/prof_sass.ncu-rep --page source --csv --print-source sass > gpurun_out/sass.csv 2>&1
  ncu -i gpurun_out/prof_sass.ncu-rep --page details > gpurun_out/prof_sass_details.txt 2>&1
  ls -la gpurun_out/prof_sass.ncu-rep
  rm -f gpurun_out/prof_sass.ncu-rep
fi
done
for what in "$@"; do
if [[ $what == ncu_lowp ]]; then
  for cfg in "c2 4" "c2 6" "c2 8"; do
    set -- $cfg
    run timeout 600 $NCU -k regex:union_kernel -s 2 -c 1 -o gpurun_out/prof_$1_p$2 \
        python -u bench.py --config $1 --p $2 --profile --no-cpu --no-e2e --no-variants --no-pipeline
    ncu -i gpurun_out/prof_$1_p$2.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_$1_p$2.csv 2>&1
    export_rep $1_p$2 prof_$1_p$2
  done
fi
done
for what in "$@"; do
if [[ $what == gthr ]]; then
  run timeout 900 python -u scripts/group_threshold.py > gpurun_out/group_threshold.log 2>&1
fi
done
for what in "$@"; do
if [[ $what == small ]]; then
  run timeout 600 python -u bench.py --config c2 --no-cpu > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.log
  run timeout 600 python -u bench.py --config c1 --no-cpu > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.log
  run timeout 600 python -u scripts/step_overhead.py > gpurun_out/step_overhead.json 2> gpurun_out/step_overhead.log
fi
done
for what in "$@"; do
if [[ $what == sanitize ]]; then
  python -u scripts/sanitize_r02.py > gpurun_out/sanitize_plain.log 2>&1; tail -1 gpurun_out/sanitize_plain.log
  for tool in memcheck racecheck synccheck; do
    run timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python -u scripts/sanitize_r02.py \
        > gpurun_out/sanitize_r02_$tool.log 2>&1
    tail -3 gpurun_out/sanitize_r02_$tool.log
  done
fi
done
for what in "$@"; do
if [[ $what == wave ]]; then
  run timeout 1500 python -u -m pytest tests/test_gpu_async_upload.py -q -x > gpurun_out/pytest_async.log 2>&1; tail -2 gpurun_out/pytest_async.log
  run timeout 600 python -u -m pytest tests/test_gpu_parity.py -q -x -k "c3_pipelined or c3_matches" > gpurun_out/pytest_c3.log 2>&1; tail -2 gpurun_out/pytest_c3.log
  run timeout 600 python -u scripts/e2e_breakdown.py > gpurun_out/e2e_breakdown.txt 2>&1
fi
done
for what in "$@"; do
if [[ $what == ncu_setup ]]; then
  run timeout 600 $NCU -k regex:build_items -c 1 -o gpurun_out/prof_build_items \
      python -u bench.py --profile --no-cpu --no-e2e --no-variants --no-pipeline
  export_rep c3_build_items prof_build_items
  run timeout 600 $NCU -k regex:run_index -c 2 -o gpurun_out/prof_run_index python -u scripts/pipeline_profile.py c3
  export_rep c3_run_index prof_run_index
fi
done
for what in "$@"; do
if [[ $what == setupcheck ]]; then
  run timeout 1500 python -u -m pytest tests/test_gpu_validation_fuzz.py tests/test_gpu_async_upload.py tests/test_gpu_parity.py -q -x -k "validation or async or interval or malformed or errors or varint or pipelined" > gpurun_out/pytest_setup.log 2>&1; tail -2 gpurun_out/pytest_setup.log
fi
done
for what in "$@"; do
if [[ $what == widened ]]; then
  for a in "c2 dense 12" "c2 interval 12" "c3 dense 12" "c3 interval 12"; do
    run timeout 900 python -u scripts/exact_bench.py $a > "gpurun_out/exact_${a// /_}.json" 2>/dev/null
  done
  run timeout 600 python -u scripts/local_metrics_bench.py c3 > gpurun_out/local_c3.json 2>/dev/null
  for tool in memcheck racecheck synccheck; do
    run timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python -u scripts/sanitize_widened.py \
        > gpurun_out/sanitizer_widened_$tool.log 2>&1
    tail -1 gpurun_out/sanitizer_widened_$tool.log
  done
fi
done
for what in "$@"; do
if [[ $what == city ]]; then
  run timeout 900 python -u scripts/city_scale.py 1650 30 12000 0 > gpurun_out/city_scale.json 2> gpurun_out/city_scale.log
  run timeout 900 python -u scripts/city_scale.py 1800 80 6500 3 > gpurun_out/city_valdivia_like.json 2> gpurun_out/city_valdivia.log
  ( time ./tools/sb_hyperball analyze 1800 1800 6500 4 16 20261017 6400 10 3 hyperball /tmp/v.csv ) \
      > gpurun_out/valdivia_like_cpp_analyze.txt 2>&1
  rm -f /tmp/v.csv
fi
done
for what in "$@"; do
if [[ $what == citysched ]]; then
  run timeout 900 python -u scripts/city_sched.py > gpurun_out/city_sched.json 2> gpurun_out/city_sched.log
fi
done
for what in "$@"; do
if [[ $what == cppanalyze ]]; then
  ( time ./tools/sb_hyperball analyze 1800 1800 6500 4 16 20261017 6400 10 3 hyperball /tmp/v.csv ) \
      > gpurun_out/valdivia_like_cpp_analyze.txt 2>&1
  ls -la /tmp/v.csv >> gpurun_out/valdivia_like_cpp_analyze.txt 2>&1; rm -f /tmp/v.csv
fi
done
for what in "$@"; do
if [[ $what == fuzz ]]; then
  run timeout 3000 python -u scripts/parity_fuzz.py 2500 2026 > gpurun_out/parity_fuzz_2500_seed2026.json 2> gpurun_out/parity_fuzz.log
fi
done
for what in "$@"; do
if [[ $what == final_checks ]]; then
  run timeout 3000 python -u scripts/parity_fuzz.py 2500 7 > gpurun_out/parity_fuzz_2500_seed7.json 2> gpurun_out/parity_fuzz7.log
  run timeout 1500 python -u scripts/determinism_c3.py > gpurun_out/determinism_c3.json 2> gpurun_out/determinism_c3.log
fi
done
for what in "$@"; do
if [[ $what == chunksweep ]]; then
  # needs the A-B build: make -B NVEXTRA=-DSB_AB_UPLOAD_CHUNKS (the product .so always uses 16 chunks)
  run timeout 1200 python -u scripts/chunk_sweep.py ${CHUNKS:-16 24 32 48 64} > gpurun_out/chunk_sweep.jsonl 2> gpurun_out/chunk_sweep.log
fi
done
for what in "$@"; do
if [[ $what == wavebug ]]; then
  run timeout 600 compute-sanitizer --tool memcheck --show-backtrace device python -u scripts/wave_fuzz.py 1 0 43 30 34 3 7 186 1218590505 10 5 > gpurun_out/wavebug_memcheck.log 2>&1
  run timeout 900 python -u scripts/wave_fuzz.py 400 11 > gpurun_out/wave_fuzz_400.log 2>&1
fi
done
for what in "$@"; do
if [[ $what == wavefix ]]; then
  run timeout 900 python -m pytest -q -x tests/test_gpu_async_upload.py > gpurun_out/pytest_async.log 2>&1
  run timeout 900 compute-sanitizer --tool memcheck python -m pytest -q -x tests/test_gpu_async_upload.py -k "overflow or fuzz_case" > gpurun_out/wavefix_memcheck.log 2>&1
  run timeout 900 python -u scripts/wave_fuzz.py 400 11 > gpurun_out/wave_fuzz_400.log 2>&1
  run timeout 3000 python -u scripts/parity_fuzz.py 2500 7 > gpurun_out/parity_fuzz_2500_seed7.json 2> gpurun_out/parity_fuzz7.log
fi
done
for what in "$@"; do
if [[ $what == e2e ]]; then
  run timeout 600 python -u scripts/e2e_breakdown.py > gpurun_out/e2e_breakdown.txt 2>&1
fi
done
for what in "$@"; do
if [[ $what == wavebig ]]; then
  run timeout 1500 python -u scripts/wave_fuzz.py 300 23 big > gpurun_out/wave_fuzz_big300.log 2>&1
fi
done
for what in "$@"; do
if [[ $what == e2e2 ]]; then
  run timeout 600 python -u scripts/e2e_breakdown.py > gpurun_out/e2e_breakdown.txt 2>&1
  run timeout 600 python -u scripts/e2e_breakdown.py > gpurun_out/e2e_breakdown_b.txt 2>&1
fi
done
for what in "$@"; do
if [[ $what == wave3 ]]; then
  run timeout 900 python -m pytest -q -x tests/test_gpu_async_upload.py > gpurun_out/pytest_async.log 2>&1
  run timeout 900 compute-sanitizer --tool memcheck python -m pytest -q -x tests/test_gpu_async_upload.py -k "growth or overflow or fuzz_case" > gpurun_out/wavefix_memcheck.log 2>&1
  run timeout 900 python -u scripts/wave_fuzz.py 400 11 > gpurun_out/wave_fuzz_400.log 2>&1
  run timeout 1500 python -u scripts/wave_fuzz.py 300 23 big > gpurun_out/wave_fuzz_big300.log 2>&1
fi
done
for what in "$@"; do
if [[ $what == fuzzbig ]]; then
  run timeout 2400 python -u scripts/parity_fuzz.py 1000 99 big > gpurun_out/parity_fuzz_big1000_seed99.json 2> gpurun_out/parity_fuzz_big.log
fi
done
for what in "$@"; do
if [[ $what == e2esmall ]]; then
  run timeout 600 python -u scripts/e2e_small.py > gpurun_out/e2e_small.txt 2>&1
fi
done
for what in "$@"; do
if [[ $what == fuzzmore ]]; then
  run timeout 1500 python -u scripts/parity_fuzz.py 2500 31337 > gpurun_out/parity_fuzz_2500_seed31337.json 2> gpurun_out/parity_fuzz31337.log
  run timeout 1500 python -u scripts/parity_fuzz.py 1000 7 big > gpurun_out/parity_fuzz_big1000_seed7.json 2> gpurun_out/parity_fuzz_big7.log
fi
done
