# Stage II: stream tests + probes (graphs on/off, pinned/device, lag / async pops)
mkdir -p gpurun_out
rm -f gpurun_out/stream_probe.log
timeout 900 python -m pytest tests -m gpu -x -q -k "stream or dropin" > gpurun_out/stream_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/stream_tests.log
for a in "" "--nographs"; do
  for d in "" "--device"; do
    for m in "--lag" "--async"; do
      timeout 300 python tools/probe_stream_pinned.py c3 300 $m $a $d >> gpurun_out/stream_probe.log 2>&1
      timeout 300 python tools/probe_stream_pinned.py c1 300 $m $a $d >> gpurun_out/stream_probe.log 2>&1
    done
  done
done
