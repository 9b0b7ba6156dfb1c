#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
for i in 1 2; do
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_$i.json 2> gpurun_out/bench_c4.err
DYCL_S2S_FUSE_LN=0 timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_nf_$i.json 2> gpurun_out/bench_c4_nf.err
done
timeout 900 python -m pytest tests/test_gpu.py -m gpu -q -k "cfg4" 2>&1 | tail -3 > gpurun_out/dev_tests.txt
for f in gpurun_out/bench_c4_*.json; do python -c "import json,sys; l=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(l['ms_per_step'],2), {k:round(v,2) for k,v in l['kernel_ms_per_step'].items()})"; done
cat gpurun_out/dev_tests.txt
