#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_multi.py -m gpu -q -x -k "device" -p no:cacheprovider 2>&1 | grep -E "Error|error|assert|FAILED" | head -20 > gpurun_out/dg2.txt
cat gpurun_out/dg2.txt
