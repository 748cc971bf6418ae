# round-end evidence: GPU tests, smoke, C3 bench (+ reference arm, launch list), every other config, stream probes
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference_arm.json 2> gpurun_out/bench_reference_arm.err; echo "ref rc=$?"
for c in c1 c2 c4 c5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"
done
rm -f gpurun_out/stream_probe.log
for cfg in c3 c1; do
  for o in "" "--packed" "--device"; do
    timeout 300 python tools/probe_stream_pinned.py $cfg 600 --async --depth 8 --push-async --wait-every 4 $o >> gpurun_out/stream_probe.log 2>&1
    timeout 300 python tools/probe_stream_pinned.py $cfg 600 --async --depth 2 --push-async $o >> gpurun_out/stream_probe.log 2>&1
    timeout 300 python tools/probe_stream_pinned.py $cfg 600 --lag $o >> gpurun_out/stream_probe.log 2>&1
  done
done
(cd /tmp && timeout 600 $GRAFT_REPO_ROOT/oracle/_ref/acceptance_b200 > $GRAFT_REPO_ROOT/gpurun_out/acceptance_b200.log 2>&1)
(cd oracle/_ref; ./bench_dropin 640 480 300 > /dev/null 2>&1; for sz in "320 240 300" "640 480 300" "1280 720 300" "1920 1088 200"; do timeout 300 ./bench_dropin $sz; done) > gpurun_out/bench_dropin.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?"
