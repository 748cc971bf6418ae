mkdir -p gpurun_out
for i in 1 2; do
STABGPU_FLAT_CHUNKS=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_flat$i.json 2>/dev/null
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_ramp$i.json 2>/dev/null
done
