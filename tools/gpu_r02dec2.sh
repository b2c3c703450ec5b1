# decoupled warp groups, second pass: group 0 throttled to half a slice ahead (mid barrier); c3 with the unscaled-A path
O=gpurun_out/r02dec2; mkdir -p $O
for c in c5 c4; do
  for dec in 0 1 2; do echo "$c decouple=$dec"; TF_EVAL_DECOUPLE=$dec timeout 300 python tools/quick_time.py $c 10 2>&1 | tail -1; done
  echo "$c decouple=1 skew=0"; TF_EVAL_SKEW_NS=0 timeout 300 python tools/quick_time.py $c 10 2>&1 | tail -1
done > $O/time.log 2>&1
for c in c3 c2; do
  echo "$c base"; timeout 300 python tools/quick_time.py $c 20 2>&1 | tail -1
  for dec in 0 1 2; do echo "$c pre0 decouple=$dec"; TF_LIB_PATH=build_u_pre0/libtf.so TF_EVAL_DECOUPLE=$dec timeout 300 python tools/quick_time.py $c 20 2>&1 | tail -1; done
  for cps in 1 2; do echo "$c pre0 decouple=1 cps=$cps"; TF_EVAL_PERSIST_CPS=$cps TF_LIB_PATH=build_u_pre0/libtf.so timeout 300 python tools/quick_time.py $c 20 2>&1 | tail -1; done
done >> $O/time.log 2>&1
cat $O/time.log | grep -v generated
