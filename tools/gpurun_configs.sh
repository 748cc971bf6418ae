# bench lines of every BASELINE config (device + e2e; CPU reference sample on c1/c2)
mkdir -p gpurun_out
for c in c1 c2 c4 c5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"
done
