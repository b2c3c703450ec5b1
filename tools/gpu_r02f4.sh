# final round-2 session (phase-2 unroll 8 at NT >= 13): smoke, all GPU tests, bench c1-c5, launch list, shard projection; PART=ncu: eval c5 + c3 captures
# projection, ncu of the evaluation and CG kernels
# (gpurun returns at most 64 MiB of gpurun_out: PART=ncu_eval5 / ncu_eval3 / ncu_cg run one full ncu capture each,
#  ~21 MB per report; PART=main everything else)
O=gpurun_out/r02f4; mkdir -p $O
if [ "$PART" != "ncu" ]; then
python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
TF_PARITY_REPORT=$O timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gputest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/gputest.log
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
# the small configs run enough steps for the clock sampler (50 ms period) to see the timed region
for cs in "c1 8000 20" "c2 4000 20" "c3 1500 10" "c4 100 5"; do set -- $cs
  timeout 900 python bench.py --config $1 --steps $2 --warmup $3 --no-stages > $O/bench_$1.json 2> $O/bench_$1.err; echo "bench $1 rc=$?"; done
timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-stages > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" --csv \
  --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-stages > $O/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 900 python tools/shard_scaling.py c5 0.05 > $O/shard.log 2>&1; echo "shard rc=$?"; tail -2 $O/shard.log | head -1
fi
if [ "$PART" = "ncu" ]; then
# (the .ncu-rep files are summarised here and deleted: gpurun returns at most 64 MiB)
for c in c5 c3; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_eval_fused -s 2 -c 1 -o $O/prof_eval_$c python tools/quick_time.py $c 2 > $O/ncu_eval_$c.log 2>&1; echo "ncu eval $c rc=$?"
  python tools/ncu_summary.py $O/prof_eval_$c.ncu-rep > $O/ncu_eval_${c}.json 2>&1
  ncu -i $O/prof_eval_$c.ncu-rep --page raw --csv > $O/ncu_eval_${c}_raw.csv 2>/dev/null
  ncu -i $O/prof_eval_$c.ncu-rep --page source --csv --print-source sass > $O/ncu_eval_${c}_source.csv 2>/dev/null
  gzip -f $O/ncu_eval_${c}_source.csv; rm -f $O/prof_eval_$c.ncu-rep
done
ls -la $O
fi
if [ "$PART" = "ncu_cg" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cg_rows -s 2 -c 1 -o $O/prof_cg_c5 python tools/time_cg.py c5 > $O/ncu_cg.log 2>&1; echo "ncu cg rc=$?"
fi
