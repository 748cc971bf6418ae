mkdir -p gpurun_out
timeout 600 python tools/probe_rgb.py 1000 > gpurun_out/probe_rgb.log 2>&1
STABGPU_RGB_ZEROCOPY=1 timeout 600 python tools/probe_rgb.py 1000 >> gpurun_out/probe_rgb.log 2>&1
timeout 600 nsys --version > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,pcie__read_bytes.sum,pcie__write_bytes.sum --clock-control none -k regex:"rgb_to_ycbcr|compose_tma" -c 6 --csv --log-file gpurun_out/rgb_ncu.csv python tools/probe_rgb.py 120 > gpurun_out/rgb_ncu.log 2>&1
