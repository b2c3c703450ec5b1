O=gpurun_out/r02l; mkdir -p $O
python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
TF_PARITY_REPORT=$O timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > $O/gputest.log 2>&1; echo "pytest rc=$?"; tail -25 $O/gputest.log
for c in c5 c4 c3 c2; do python tools/time_cg.py $c; done
