#!/bin/bash
# One GPU session: tests, bench, ncu launch list + full capture of the fused kernel.
# usage: tools/gpu_round.sh [tag] [stages...]   stages: test bench ncu full
set -u
TAG=${1:-r01}; shift || true
STAGES=${@:-test bench ncu full}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_$TAG.txt 2>&1
for s in $STAGES; do
  case $s in
    test)
      python __graft_entry__.py smoke > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
      timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gputest_$TAG.log 2>&1; echo "pytest-gpu rc=$?"; tail -5 gpurun_out/gputest_$TAG.log ;;
    bench)
      timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench_$TAG.json; tail -3 gpurun_out/bench_$TAG.err ;;
    ncu)
      timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-stages > gpurun_out/plain_$TAG.log 2>&1 && \
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" --csv \
        --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-stages > gpurun_out/ncu_$TAG.log 2>&1
      echo "ncu launches rc=$?"; tail -2 gpurun_out/launches_$TAG.csv ;;
    full)
      CFG=${NCU_CFG:-c5}
      timeout 600 python tools/quick_time.py $CFG 2 > gpurun_out/qt_$TAG.log 2>&1 && \
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_eval_fused -s 2 -c 1 \
        -o gpurun_out/prof_${CFG}_$TAG python tools/quick_time.py $CFG 2 > gpurun_out/ncufull_$TAG.log 2>&1
      echo "ncu full rc=$?"; tail -3 gpurun_out/ncufull_$TAG.log ;;
    fullgemm)
      timeout 600 python tools/time_compress.py c5 1 > gpurun_out/tc_$TAG.log 2>&1 && \
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_dmma -s 0 -c 1 \
        -o gpurun_out/prof_gram_c5_$TAG python tools/time_compress.py c5 1 > gpurun_out/ncugemm_$TAG.log 2>&1
      echo "ncu gemm rc=$?"; tail -3 gpurun_out/ncugemm_$TAG.log ;;
    quick)
      for c in c2 c3 c4 c5; do timeout 300 python tools/quick_time.py $c 5 2>&1 | tail -1; done ;;
  esac
done
