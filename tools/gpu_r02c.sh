# CG rework check: parity of the CG/matvec tests, then timings of both kernels with the stage timeline
O=gpurun_out/r02c; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cg or matvec or dgn" -p no:cacheprovider > $O/t_parity.log 2>&1; echo "parity rc=$?"; tail -3 $O/t_parity.log
TF_PARITY_REPORT=$O timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "cg" -p no:cacheprovider > $O/t_full.log 2>&1; echo "full rc=$?"; tail -3 $O/t_full.log
for c in c5 c4 c3 c2; do python tools/time_cg.py $c; TF_CG_KERNEL=grid python tools/time_cg.py $c; TF_CG_TSTAMP=1 python tools/time_cg.py $c | tail -3; done
