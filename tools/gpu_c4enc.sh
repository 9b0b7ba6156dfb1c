#!/bin/bash
# cfg4: encoder LayerNorms fused into the out-proj / FFN-down GEMMs (multi-round persistent grid) A/B; tests
mkdir -p gpurun_out
rm -f gpurun_out/c4enc_*.json
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
for i in 1 2; do
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c4enc_on_$i.json 2> gpurun_out/c4enc.err
DYCL_S2S_FUSE_LN=0 timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c4enc_off_$i.json 2>> gpurun_out/c4enc.err
done
timeout 900 python -m pytest tests -m gpu -q -k "cfg4 or s2s or seq2seq or conv_kernel" 2>&1 | tail -3 > gpurun_out/c4enc_tests.txt
for f in gpurun_out/c4enc_*.json; do python -c "import json,sys; l=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(l['ms_per_step'],2), {k:round(v,2) for k,v in l.get('kernel_ms_per_step',{}).items()})"; done
cat gpurun_out/c4enc_tests.txt; tail -3 gpurun_out/c4enc.err
