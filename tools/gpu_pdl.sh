#!/bin/bash
# PDL on the image graphs (conv / GEMM / compaction kernels): A/B cfg2, cfg3, cfg5; full GPU tests
mkdir -p gpurun_out
rm -f gpurun_out/pdl_*.json
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
for c in 2 3; do for i in 1 2; do
timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/pdl_on_c${c}_$i.json 2> gpurun_out/pdl.err
DYCL_PDL=0 timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/pdl_off_c${c}_$i.json 2>> gpurun_out/pdl.err
done; done
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/pdl_on_c5_1.json 2>> gpurun_out/pdl.err
DYCL_PDL=0 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/pdl_off_c5_1.json 2>> gpurun_out/pdl.err
for f in gpurun_out/pdl_*.json; do python -c "import json,sys; l=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(l['ms_per_step'],4), l['clocks']['sm_mhz'])"; done
tail -3 gpurun_out/pdl.err
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3
