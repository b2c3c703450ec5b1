# final round-2 session: smoke, all GPU tests, bench (ours + reference), launch list, shard projection, CG ncu
O=gpurun_out/r02final; mkdir -p $O
python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
TF_PARITY_REPORT=$O timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gputest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/gputest.log
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-stages > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" --csv \
  --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-stages > $O/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 900 python tools/shard_scaling.py c5 0.05 > $O/shard.log 2>&1; echo "shard rc=$?"; tail -2 $O/shard.log | head -1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cg_rows -s 2 -c 1 -o $O/prof_cg_c5 python tools/time_cg.py c5 > $O/ncu_cg.log 2>&1; echo "ncu cg rc=$?"
