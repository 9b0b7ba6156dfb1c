#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
for i in 1 2 3; do
timeout 600 python -m pytest tests/test_gpu_multi.py -m gpu -q -x -k "cfg5" 2>&1 | grep -v "^$" | tail -15 > gpurun_out/dev_multi_$i.txt
tail -2 gpurun_out/dev_multi_$i.txt
done
DYCL_CONV_DBG=16777216 timeout 600 python -m pytest tests/test_gpu_multi.py -m gpu -q -x -k "cfg5" 2>&1 | tail -2
