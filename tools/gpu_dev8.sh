#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
timeout 600 python -m pytest tests/test_gpu.py -m gpu -q -x -k "nhwc" 2>&1 | tail -5 > gpurun_out/dev_conv.txt
cat gpurun_out/dev_conv.txt | tail -3
timeout 300 python tools/step_profile5.py 2048 2 > gpurun_out/prof5.json 2> gpurun_out/prof5.err
timeout 1500 python -m pytest tests/test_gpu.py tests/test_gpu_edge.py -m gpu -q -k "cfg5" 2>&1 | tail -5 > gpurun_out/dev_tests.txt
cat gpurun_out/dev_tests.txt | tail -2
