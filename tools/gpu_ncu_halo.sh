#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
DYCL_GRAPH=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_conv_halo -c 2 \
   -o gpurun_out/c5_halo3_full python tools/ncu_chunk.py 5 2048 > gpurun_out/c5_halo3_full.out 2>&1
timeout 900 python tools/ab5p.py 2048 2 > gpurun_out/ab5.txt 2>&1
