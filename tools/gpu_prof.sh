#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu.py -m gpu -q -x -k "cfg5 or rebalance" 2>&1 | tail -3 > gpurun_out/dev_tests.txt
timeout 300 python tools/step_profile5.py 2048 2 > gpurun_out/prof5.json 2> gpurun_out/prof5.err
bash tools/profile_r02.sh > gpurun_out/profile_r02.log 2>&1
cat gpurun_out/dev_tests.txt
