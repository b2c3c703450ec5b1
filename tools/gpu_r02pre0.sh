# unscaled-A/TMEM Pi pass at every R, decoupling only at NT = 3, two CTAs per SM for NT <= 3: timing + all GPU tests
O=gpurun_out/r02pre0; mkdir -p $O
for c in c3 c4 c5; do timeout 300 python tools/quick_time.py $c 20 2>&1 | tail -1; done > $O/time.log 2>&1
for R in 8 16 24 32; do timeout 300 python tools/time_eval_dims.py 500 500 500 $R 20 2>&1 | tail -1; done >> $O/time.log 2>&1
cat $O/time.log
python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gputest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/gputest.log
