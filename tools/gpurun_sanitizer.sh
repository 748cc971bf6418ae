# compute-sanitizer memcheck over a subset of the GPU parity tests ($K), then racecheck over a smaller one ($KR)
mkdir -p gpurun_out
K=${K:-"short_clip or stream_equals_stage1 or streams_equal or sharded_equals or sequence_420 or rgb_equals_planes"}
KR=${KR:-"short_clip"}
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 3 --print-limit 20 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/sanitizer_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/sanitizer_memcheck.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 3 --print-limit 20 python -m pytest tests -m gpu -x -q -k "$KR" > gpurun_out/sanitizer_racecheck.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/sanitizer_racecheck.log
tail -5 gpurun_out/sanitizer_memcheck.log gpurun_out/sanitizer_racecheck.log
