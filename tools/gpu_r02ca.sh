mkdir -p gpurun_out/r02ca
for c in c5 c4 c3 c2; do timeout 300 python tools/quick_time.py $c 10 2>&1 | tail -3; done > gpurun_out/r02ca/time.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -x -q -m gpu > gpurun_out/r02ca/pytest.log 2>&1; echo pytest rc=$? >> gpurun_out/r02ca/pytest.log
