# Pi-form k-step loop unroll above NT = 8 (A: phase 2 by 8; B: phase 2 by 2; C: both by 8; D: phase 2 by 8 and
# phase 3 by 4; E: phase 3 by 8) against full unroll (the in-tree build), c5 (NT 13) and 500^3 at R = 72 / 120
O=gpurun_out/r02unr; mkdir -p $O
for rep in 1 2; do
  echo "c5 base"; timeout 300 python tools/quick_time.py c5 10 2>&1 | tail -1
  for v in A B C D E; do echo "c5 $v"; TF_LIB_PATH=build_u_$v/libtf.so timeout 300 python tools/quick_time.py c5 10 2>&1 | tail -1; done
done > $O/time.log 2>&1
for R in 72 120; do
  echo "R=$R base"; timeout 300 python tools/time_eval_dims.py 500 500 500 $R 10 2>&1 | tail -1
  for v in A C D E; do echo "R=$R $v"; TF_LIB_PATH=build_u_$v/libtf.so timeout 300 python tools/time_eval_dims.py 500 500 500 $R 10 2>&1 | tail -1; done
done >> $O/time.log 2>&1
grep -v generated $O/time.log
