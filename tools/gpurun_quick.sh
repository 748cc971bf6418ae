# quick loop: the GPU parity tests matching $K (default: all) + one C3 bench line
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q ${K:+-k "$K"} > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline ${ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
