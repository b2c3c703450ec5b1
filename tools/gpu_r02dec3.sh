# c3 (R = 20): prescaled (kPre) vs unscaled-A/TMEM Pi pass, decoupled groups, CTAs per SM, skew
O=gpurun_out/r02dec3; mkdir -p $O
for cps in 1 2; do echo "c3 base cps=$cps"; TF_EVAL_PERSIST_CPS=$cps timeout 300 python tools/quick_time.py c3 50 2>&1 | tail -1; done > $O/time.log 2>&1
for cps in 1 2; do for dec in 0 1 2; do for sk in 0 520; do
  echo "c3 pre0 cps=$cps dec=$dec skew=$sk"; TF_LIB_PATH=build_u_pre0/libtf.so TF_EVAL_PERSIST_CPS=$cps TF_EVAL_DECOUPLE=$dec TF_EVAL_SKEW_NS=$sk timeout 300 python tools/quick_time.py c3 50 2>&1 | tail -1
done; done; done >> $O/time.log 2>&1
echo "c3 pre0 default"; TF_LIB_PATH=build_u_pre0/libtf.so timeout 300 python tools/quick_time.py c3 50 2>&1 | tail -1 >> $O/time.log
python - >> $O/time.log 2>&1 <<'PY'
import ctypes, torch
for lib in ["paper_2110_05997_b200/libtf.so", "build_u_pre0/libtf.so"]:
    print(lib)
PY
cat $O/time.log | grep -v generated
