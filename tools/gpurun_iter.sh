# one iteration: GPU tests matching $K (default all), stream probes, C3 + C1 bench lines
mkdir -p gpurun_out
rm -f gpurun_out/stream_probe.log
timeout 1500 python -m pytest tests -m gpu -x -q ${K:+-k "$K"} > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
for d in "" "--device"; do
  for m in "--lag" "--async"; do
    timeout 300 python tools/probe_stream_pinned.py c3 300 $m $d >> gpurun_out/stream_probe.log 2>&1
    timeout 300 python tools/probe_stream_pinned.py c1 300 $m $d >> gpurun_out/stream_probe.log 2>&1
  done
done
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --config c1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo "bench c1 rc=$?"
