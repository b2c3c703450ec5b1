# decoupled warp groups in the Pi-form pass: timing against the per-slice block barrier, skew sweep, then parity
O=gpurun_out/r02dec; mkdir -p $O
for c in c5 c4; do
  for dec in 0 1; do echo "$c decouple=$dec"; TF_EVAL_DECOUPLE=$dec timeout 300 python tools/quick_time.py $c 10 2>&1 | tail -1; done
done > $O/time.log 2>&1
for sk in 0 1000 2000 5000; do echo "c5 skew=$sk"; TF_EVAL_SKEW_NS=$sk timeout 300 python tools/quick_time.py c5 10 2>&1 | tail -1; done >> $O/time.log 2>&1
for sk in 0 1000 3000; do echo "c4 skew=$sk"; TF_EVAL_SKEW_NS=$sk timeout 300 python tools/quick_time.py c4 10 2>&1 | tail -1; done >> $O/time.log 2>&1
cat $O/time.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py tests/test_gpu_fullsize.py -x -q -m gpu > $O/pytest.log 2>&1; echo pytest rc=$? >> $O/pytest.log; tail -3 $O/pytest.log
