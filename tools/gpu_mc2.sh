#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
timeout 600 python -m pytest tests/test_gpu.py -m gpu -q -k "multicast or (conv_kernel and tma)" 2>&1 | tail -2
for i in 1 2; do
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/mc2_$i.json 2> gpurun_out/mc2.err
done
for f in gpurun_out/mc2_*.json; do python -c "import json,sys; l=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(l['ms_per_step'],2))"; done
