#!/bin/bash
# fused LayerNorm partials through DSMEM (cluster of the M tile's N tiles) vs L2 counter; cfg4 tests
mkdir -p gpurun_out
rm -f gpurun_out/lnc_*.json
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
for i in 1 2; do
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/lnc_on_$i.json 2> gpurun_out/lnc.err
DYCL_LN_CLUSTER=0 timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/lnc_off_$i.json 2>> gpurun_out/lnc.err
done
for f in gpurun_out/lnc_*.json; do python -c "import json,sys; l=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(l['ms_per_step'],2))"; done
tail -3 gpurun_out/lnc.err
timeout 900 python -m pytest tests -m gpu -q -k "cfg4 or s2s or seq2seq or conv_kernel" 2>&1 | tail -2
