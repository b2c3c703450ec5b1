# guards, bench (ours + reference), launch list, full ncu of the two hot kernels at c5
O=gpurun_out/r02n; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_guards.py -q -p no:cacheprovider > $O/guards.log 2>&1; echo "guards rc=$?"; tail -3 $O/guards.log
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; tail -c 600 $O/bench.json; tail -2 $O/bench.err
timeout 900 python bench.py --impl reference > $O/ref.json 2> $O/ref.err; echo "ref rc=$?"; tail -c 400 $O/ref.json
timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-stages > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" --csv \
  --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-stages > $O/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 600 python tools/quick_time.py c5 2 > $O/qt.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_eval_fused -s 2 -c 1 -o $O/prof_eval_c5 python tools/quick_time.py c5 2 > $O/ncu_eval.log 2>&1; echo "ncu eval rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cg_rows -s 2 -c 1 -o $O/prof_cg_c5 python tools/time_cg.py c5 > $O/ncu_cg.log 2>&1; echo "ncu cg rc=$?"
