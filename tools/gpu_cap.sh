#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_caption.py tests/test_abi.py -q -x -s 2>&1 | grep -v "^$" | tail -30 > gpurun_out/dev_cap.txt
timeout 900 python -m pytest tests/test_gpu.py -m gpu -q -k "cfg2_sdn or cfg3_skip" 2>&1 | tail -3 >> gpurun_out/dev_cap.txt
cat gpurun_out/dev_cap.txt | tail -25
