# edge-tile k-step skipping: timing, then the parity / guard suites
mkdir -p gpurun_out/r02es
for c in c5 c4 c3 c2; do timeout 300 python tools/quick_time.py $c 10 2>&1 | tail -1; done > gpurun_out/r02es/time.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -x -q -m gpu > gpurun_out/r02es/pytest.log 2>&1; echo pytest rc=$? >> gpurun_out/r02es/pytest.log
