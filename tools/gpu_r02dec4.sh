# small-R Pi pass: prescaled (base) vs unscaled-A/TMEM (pre0) x decoupled x CTAs per SM, R = 8..40 at 500^3
O=gpurun_out/r02dec4; mkdir -p $O
for R in 8 16 24 32 40; do
  for cps in 0 1 2; do
    echo "R=$R base cps=$cps"; TF_EVAL_PERSIST_CPS=$cps timeout 300 python tools/time_eval_dims.py 500 500 500 $R 20 2>&1 | tail -1
    for dec in 0 2; do echo "R=$R pre0 cps=$cps dec=$dec"; TF_LIB_PATH=build_u_pre0/libtf.so TF_EVAL_PERSIST_CPS=$cps TF_EVAL_DECOUPLE=$dec timeout 300 python tools/time_eval_dims.py 500 500 500 $R 20 2>&1 | tail -1; done
  done
done > $O/time.log 2>&1
cat $O/time.log
