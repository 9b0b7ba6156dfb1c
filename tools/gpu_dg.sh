#!/bin/bash
# device-rebalanced runs through the captured-graph path: multi tests twice + cfg4 quick bench
mkdir -p gpurun_out
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
: > gpurun_out/dg.txt
for i in 1 2; do
  timeout 600 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider 2>&1 | tail -1 >> gpurun_out/dg.txt
done
DYCL_GRAPH=0 timeout 600 python -m pytest tests/test_gpu_multi.py -m gpu -q -k device -p no:cacheprovider 2>&1 | tail -1 >> gpurun_out/dg.txt
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/dg_c4.json 2>> gpurun_out/dg.txt
python -c "import json; l=json.loads(open('gpurun_out/dg_c4.json').read().strip().splitlines()[-1]); print('cfg4', round(l['ms_per_step'],2))" >> gpurun_out/dg.txt
cat gpurun_out/dg.txt
