#!/bin/bash
# cfg5 zero-copy stage entries: bitwise test, cfg5 parity, A/B chunk timing (28x28 entry on/off)
mkdir -p gpurun_out
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu.py -m gpu -q -s -k "cfg5" 2>&1 | grep -v "^$" | tail -8 > gpurun_out/zc_tests.txt
for i in 1 2; do
DYCL_ZC_PROJ_MIN=4 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/zc_new_$i.json 2> gpurun_out/zc.err
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/zc_old_$i.json 2>> gpurun_out/zc.err
done
for f in gpurun_out/zc_*.json; do python -c "import json,sys; l=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(l['ms_per_step'],2), l['clocks']['sm_mhz'], {k:round(v,2) for k,v in l.get('kernel_ms_per_step',{}).items()})"; done
cat gpurun_out/zc_tests.txt
