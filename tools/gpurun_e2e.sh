# e2e chunk shapes on the small-frame configs
mkdir -p gpurun_out
for c in c2 c5; do
for cf in noramp default; do
  if [ $cf = default ]; then unset STABGPU_NO_FLAT_RAMP; else export STABGPU_NO_FLAT_RAMP=1; fi
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/e2e_${c}_$cf.json 2> gpurun_out/e2e_${c}_$cf.err; echo "bench $c $cf rc=$?"
done; done
unset STABGPU_NO_FLAT_RAMP
timeout 1200 python -m pytest tests -m gpu -x -q -k "host or chunk or sequence or config" > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
