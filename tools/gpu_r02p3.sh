# phase-3 (tensor-memory) k-step loop unrolled by 8 at every NT (build_u_J) vs the in-tree build
O=gpurun_out/r02p3; mkdir -p $O
for rep in 1 2; do for c in c4 c5; do
  echo "$c base"; timeout 300 python tools/quick_time.py $c 10 2>&1 | tail -1
  echo "$c J"; TF_LIB_PATH=build_u_J/libtf.so timeout 300 python tools/quick_time.py $c 10 2>&1 | tail -1
done; done > $O/time.log 2>&1
for R in 40 72; do
  echo "R=$R base"; timeout 300 python tools/time_eval_dims.py 500 500 500 $R 10 2>&1 | tail -1
  echo "R=$R J"; TF_LIB_PATH=build_u_J/libtf.so timeout 300 python tools/time_eval_dims.py 500 500 500 $R 10 2>&1 | tail -1
done >> $O/time.log 2>&1
grep -v generated $O/time.log
