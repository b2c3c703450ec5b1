set -u
O=gpurun_out/r02a; mkdir -p $O
nproc > $O/host.txt; lscpu | grep -E "Model name|^CPU\(s\)|Socket|Thread" >> $O/host.txt; free -g >> $O/host.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv >> $O/host.txt
python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?"
TF_PARITY_REPORT=$O timeout 3000 python -m pytest tests -m gpu -q --durations=40 -p no:cacheprovider > $O/gputest.log 2>&1; echo "pytest rc=$?"
tail -60 $O/gputest.log
for c in c1 c2 c3 c4; do timeout 300 python tools/quick_time.py $c 10 2>&1 | tail -1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_eval_fused -s 2 -c 1 -o $O/prof_c3 python tools/quick_time.py c3 2 > $O/ncufull_c3.log 2>&1; echo "ncu rc=$?"
