#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
timeout 600 python -m pytest tests/test_gpu.py -m gpu -q -x -k "nhwc" 2>&1 | tail -5 > gpurun_out/dev_conv.txt
cat gpurun_out/dev_conv.txt | tail -3
timeout 900 python tools/ab5p.py 2048 6 DYCL_CONV_DBG=8388608 > gpurun_out/ab5.txt 2>&1
cat gpurun_out/ab5.txt
