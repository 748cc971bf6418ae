mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "stream or dropin or tracker" > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
rm -f gpurun_out/stream_probe.log
for i in 1 2; do
for m in "--lag" "--async" "--async --push-async" "--lag --push-async" "--async --depth 3 --push-async"; do
    timeout 300 python tools/probe_stream_pinned.py c3 300 $m >> gpurun_out/stream_probe.log 2>&1
    timeout 300 python tools/probe_stream_pinned.py c1 300 $m >> gpurun_out/stream_probe.log 2>&1
done; done
