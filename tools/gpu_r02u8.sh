# phase-2 k-loop unroll 8 for NT >= 13 (in-tree build): timing, GPU tests, c5 bench
O=gpurun_out/r02u8; mkdir -p $O
for rep in 1 2; do timeout 300 python tools/quick_time.py c5 10 2>&1 | tail -1; done > $O/time.log 2>&1
for R in 104 112 128; do timeout 300 python tools/time_eval_dims.py 500 500 500 $R 10 2>&1 | tail -1; done >> $O/time.log 2>&1
grep -v generated $O/time.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gputest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/gputest.log
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; tail -1 $O/bench.json | cut -c1-300
