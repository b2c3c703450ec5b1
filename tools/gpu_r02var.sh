# compiler-level variants of the Pi pass (phase fence between phase 3 and phase 2; phase-2 k-loop unroll 4 / 8)
O=gpurun_out/r02var; mkdir -p $O
for rep in 1 2; do
for c in c5 c4; do
  echo "$c base"; timeout 300 python tools/quick_time.py $c 10 2>&1 | tail -1
  for v in fence u4 u8; do echo "$c $v"; TF_LIB_PATH=build_u_$v/libtf.so timeout 300 python tools/quick_time.py $c 10 2>&1 | tail -1; done
done; done > $O/time.log 2>&1
grep -v generated $O/time.log
