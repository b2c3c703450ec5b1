O=gpurun_out/${TAG:-r02f}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cg or matvec or dgn" -p no:cacheprovider > $O/t_parity.log 2>&1; echo "parity rc=$?"; tail -2 $O/t_parity.log
for c in c5 c4 c3; do python tools/time_cg.py $c; TF_CG_TSTAMP=1 python tools/time_cg.py $c | tail -3; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cg_rows -s 2 -c 1 -o $O/prof_cgrows_c5 python tools/time_cg.py c5 > $O/ncu.log 2>&1; echo ncu rc=$?
