#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
tail -3 gpurun_out/build.txt
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -s 2>&1 | grep -v "^$" | tail -25 > gpurun_out/dev_drb.txt
cat gpurun_out/dev_drb.txt
