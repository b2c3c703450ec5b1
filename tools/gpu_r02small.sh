# bench lines of c1-c4 with clock samples (steps sized for the 50 ms sampler)
O=gpurun_out/r02final; mkdir -p $O
for cs in "c1 8000 20" "c2 4000 20" "c3 1500 10" "c4 100 5"; do set -- $cs
  timeout 900 python bench.py --config $1 --steps $2 --warmup $3 --no-stages > $O/bench_$1.json 2> $O/bench_$1.err; echo "bench $1 rc=$?"; done
