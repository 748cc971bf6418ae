# detection loop: detection / config parity / stream tests, C1 + C3 + C2 bench lines, stream probes
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "detect or corner or config or stream" > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
for c in c1 c3 c2; do
timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"
done
rm -f gpurun_out/stream_probe.log
for m in "--lag" "--async"; do
  timeout 300 python tools/probe_stream_pinned.py c3 300 $m --device >> gpurun_out/stream_probe.log 2>&1
  timeout 300 python tools/probe_stream_pinned.py c1 300 $m --device >> gpurun_out/stream_probe.log 2>&1
done
