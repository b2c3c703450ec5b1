O=gpurun_out/r02o; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_guards.py -q -p no:cacheprovider > $O/guards.log 2>&1; echo "guards rc=$?"; tail -3 $O/guards.log
timeout 900 python tools/shard_scaling.py c5 0.05 > $O/shard.log 2>&1; echo "shard rc=$?"; tail -5 $O/shard.log
for c in c1 c2 c3 c4; do timeout 900 python bench.py --config $c --no-stages > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench $c rc=$?"; done
