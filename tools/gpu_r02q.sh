O=gpurun_out/r02q; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_als.py -q -p no:cacheprovider -k c5 > $O/als.log 2>&1; echo "als rc=$?"; tail -2 $O/als.log
timeout 900 python bench.py --config c1 --steps 8000 --warmup 20 --no-stages > $O/bench_c1.json 2> $O/bench_c1.err; echo "c1 rc=$?"
timeout 900 python bench.py --config c2 --steps 4000 --warmup 20 --no-stages > $O/bench_c2.json 2> $O/bench_c2.err; echo "c2 rc=$?"
timeout 900 python bench.py --config c3 --steps 1500 --warmup 10 --no-stages > $O/bench_c3.json 2> $O/bench_c3.err; echo "c3 rc=$?"
timeout 900 python bench.py --config c4 --steps 100 --warmup 5 --no-stages > $O/bench_c4.json 2> $O/bench_c4.err; echo "c4 rc=$?"
