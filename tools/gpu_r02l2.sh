# DRAM bytes of the evaluation kernel: 4-D TMA view (no padding-row over-read) x L2 promotion; then parity
O=gpurun_out/r02l2; mkdir -p $O
for t4 in 1 0; do for pr in 0 256; do
  echo "tma4=$t4 promo=$pr"
  TF_EVAL_TMA4=$t4 TF_EVAL_L2PROMO=$pr timeout 300 python tools/quick_time.py c5 10 2>&1 | tail -1
  TF_EVAL_TMA4=$t4 TF_EVAL_L2PROMO=$pr timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:k_eval_fused -s 2 -c 1 python tools/quick_time.py c5 1 2>&1 | grep -E "dram__"
done; done > $O/l2.log 2>&1
for c in c4 c3; do timeout 300 python tools/quick_time.py $c 10 2>&1 | tail -1; done >> $O/l2.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -x -q -m gpu > $O/pytest.log 2>&1; echo pytest rc=$? >> $O/pytest.log
