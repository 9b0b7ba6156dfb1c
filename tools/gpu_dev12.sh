#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu.py tests/test_gpu_edge.py tests/test_gpu_multi.py -m gpu -q -x -k "cfg5 or nhwc" 2>&1 | tail -5 > gpurun_out/dev_tests.txt
cat gpurun_out/dev_tests.txt | tail -3
timeout 600 python -m pytest tests/test_gpu_multi.py -m gpu -q -x -k "cfg5" 2>&1 | tail -2
timeout 900 python tools/ab5p.py 2048 6 > gpurun_out/ab5.txt 2>&1
cat gpurun_out/ab5.txt
