# one ncu --set full capture of the hot kernels of the C3 bench step (bench itself must exit 0 first)
mkdir -p gpurun_out
K=${K:-'regex:compose_tma|lk_chain|resp_stream'}
timeout 1200 ncu --set full --clock-control none --import-source on -k "$K" -c ${C:-4} \
  -o gpurun_out/${OUT:-ncu_full} -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline ${ARGS:-} > gpurun_out/${OUT:-ncu_full}.log 2>&1
echo "ncu rc=$?"
