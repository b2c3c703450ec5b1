# CG with the scalar exchange ring (alpha, beta without grid barriers): timing + CG parity
O=gpurun_out/r02ring; mkdir -p $O
for c in c5 c4 c3 c2; do timeout 300 python tools/time_cg.py $c 2>&1 | tail -2; done > $O/t.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -x -q -m gpu -k "cg or matvec or dgn" > $O/pytest.log 2>&1; echo pytest rc=$? >> $O/pytest.log

