# phase-2 B fragments as 16-byte pairs (TF_B_PAIR=1, the in-tree build) vs single 8-byte loads (build_u_pair0)
O=gpurun_out/r02pair; mkdir -p $O
for rep in 1 2; do
for c in c5 c4 c3; do
  echo "$c pair=1"; timeout 300 python tools/quick_time.py $c 10 2>&1 | tail -1
  echo "$c pair=0"; TF_LIB_PATH=build_u_pair0/libtf.so timeout 300 python tools/quick_time.py $c 10 2>&1 | tail -1
done; done > $O/time.log 2>&1
for R in 8 16 32 40 64 120; do
  echo "R=$R pair=1"; timeout 300 python tools/time_eval_dims.py 500 500 500 $R 10 2>&1 | tail -1
  echo "R=$R pair=0"; TF_LIB_PATH=build_u_pair0/libtf.so timeout 300 python tools/time_eval_dims.py 500 500 500 $R 10 2>&1 | tail -1
done >> $O/time.log 2>&1
grep -v generated $O/time.log
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -x -q -m gpu > $O/pytest.log 2>&1; echo pytest rc=$? >> $O/pytest.log; tail -3 $O/pytest.log
