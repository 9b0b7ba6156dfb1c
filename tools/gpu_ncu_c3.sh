#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
DYCL_GRAPH=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_conv_gemm -s 3 -c 1 \
   -o gpurun_out/c5_conv3_full python tools/ncu_chunk.py 5 2048 > gpurun_out/c5_conv3_full.out 2>&1
ls -la gpurun_out/c5_conv3_full.ncu-rep
