#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
timeout 900 python tools/ab5p.py 2048 8 DYCL_HALO_KSKIP=0 DYCL_CONV_DBG=8388608 > gpurun_out/ab5.txt 2>&1
cat gpurun_out/ab5.txt
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_throttle_reasons.active --format=csv
