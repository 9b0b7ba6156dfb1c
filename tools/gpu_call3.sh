#!/bin/bash
# cfg4 launch list + ncu --set full on the decode kernels
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s2s_launches.csv python tools/s2s_probe.py 1024 1 > gpurun_out/s2s_probe.log 2>&1
echo "launch list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_attn_decoder -c 2 -o gpurun_out/s2s_attn -f python tools/s2s_probe.py 1024 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_layernorm -s 20 -c 1 -o gpurun_out/s2s_ln -f python tools/s2s_probe.py 1024 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tma -s 40 -c 8 -o gpurun_out/s2s_gemm -f python tools/s2s_probe.py 1024 1 > /dev/null 2>&1
ls -la gpurun_out/
