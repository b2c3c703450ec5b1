for c in c4 c5 c3; do
  for ks in 0 1 2 3 4 5 6 8; do echo "ks=$ks"; TF_EVAL_KSPLIT=$ks timeout 300 python tools/quick_time.py $c 10 2>&1 | tail -1; done
  for ov in 0.5 1 4 8; do echo "ovh=$ov"; TF_EVAL_KSPLIT_OVH=$ov timeout 300 python tools/quick_time.py $c 10 2>&1 | tail -1; done
done
