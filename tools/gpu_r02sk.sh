# stream-K evaluation: timing with and without, CTAs per SM of the persistent grid, then the parity / guard suites
mkdir -p gpurun_out/r02sk
for c in c3 c5 c4 c2 c1; do
  for sk in 1 0; do echo "streamk=$sk"; TF_EVAL_STREAMK=$sk timeout 300 python tools/quick_time.py $c 10 2>&1 | tail -1; done
done > gpurun_out/r02sk/time.log 2>&1
for cps in 1 2 3; do echo "c3 cps=$cps"; TF_EVAL_PERSIST_CPS=$cps timeout 300 python tools/quick_time.py c3 10 2>&1 | tail -1; done >> gpurun_out/r02sk/time.log 2>&1
for cps in 1 2; do echo "c2 cps=$cps"; TF_EVAL_PERSIST_CPS=$cps timeout 300 python tools/quick_time.py c2 10 2>&1 | tail -1; done >> gpurun_out/r02sk/time.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -x -q -m gpu > gpurun_out/r02sk/pytest.log 2>&1; echo pytest rc=$? >> gpurun_out/r02sk/pytest.log
