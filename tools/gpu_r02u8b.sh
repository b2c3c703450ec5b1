# NT = 13/14/16 with the phase-2 unroll 8 (in-tree) vs full unroll (build_u_full), same box
O=gpurun_out/r02u8b; mkdir -p $O
for rep in 1 2; do for R in 104 112 128; do
  echo "R=$R u8"; timeout 300 python tools/time_eval_dims.py 500 500 500 $R 10 2>&1 | tail -1
  echo "R=$R full"; TF_LIB_PATH=build_u_full/libtf.so timeout 300 python tools/time_eval_dims.py 500 500 500 $R 10 2>&1 | tail -1
done; done > $O/time.log 2>&1
for lib in paper_2110_05997_b200/libtf.so build_u_full/libtf.so; do echo "c5 $lib"; TF_LIB_PATH=$lib timeout 300 python tools/quick_time.py c5 10 2>&1 | tail -1; done >> $O/time.log 2>&1
grep -v generated $O/time.log
