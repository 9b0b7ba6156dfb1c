#!/bin/bash
# device-rebalancing in-process tests, repeated (lazy-loading deadlock fix), then the full multi file
mkdir -p gpurun_out
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
: > gpurun_out/multi_rep.txt
for i in 1 2 3; do
  timeout 600 python -m pytest tests/test_gpu_multi.py -m gpu -q -k "device" -p no:cacheprovider 2>&1 | tail -1 >> gpurun_out/multi_rep.txt
done
timeout 600 python -m pytest tests/test_gpu_multi.py tests/test_gpu_edge.py -m gpu -q -p no:cacheprovider 2>&1 | tail -2 >> gpurun_out/multi_rep.txt
cat gpurun_out/multi_rep.txt
