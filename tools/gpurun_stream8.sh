# full GPU tests, then Stage II probes: caller 8 frames ahead, planes in three arrays or one planar buffer per frame
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
rm -f gpurun_out/stream_probe.log
for cfg in c3 c1; do
  for o in "" "--packed" "--device"; do
    timeout 300 python tools/probe_stream_pinned.py $cfg 600 --async --depth 8 --push-async --wait-every 4 $o >> gpurun_out/stream_probe.log 2>&1
    timeout 300 python tools/probe_stream_pinned.py $cfg 600 --async --depth 2 --push-async $o >> gpurun_out/stream_probe.log 2>&1
    timeout 300 python tools/probe_stream_pinned.py $cfg 600 --lag $o >> gpurun_out/stream_probe.log 2>&1
  done
done
tail -3 gpurun_out/gpu_tests.log; cat gpurun_out/stream_probe.log
