# LK loop: tracking / sequence / config parity tests, C3 + C4 bench lines
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "track or lk or weed or sequence or config or stream or sharded" > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
for c in c3 c4; do
timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"
done
