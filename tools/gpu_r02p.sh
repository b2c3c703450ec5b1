O=gpurun_out/${TAG:-r02p}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -q -x -k "cg or matvec or dgn or guard" -p no:cacheprovider > $O/t.log 2>&1; echo "tests rc=$?"; tail -2 $O/t.log
for c in c5 c4 c3 c2; do python tools/time_cg.py $c; done
TF_CG_TSTAMP=1 python tools/time_cg.py c5 | tail -3
