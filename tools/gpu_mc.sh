#!/bin/bash
# k_gemm_tma CTA pairs with multicast W (BN=256 GEMMs): A/B on cfg4 + GEMM-path tests
mkdir -p gpurun_out
rm -f gpurun_out/mc_*.json
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "conv_kernel and 1536" 2>&1 | tail -2
for i in 1 2; do
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/mc_on_$i.json 2> gpurun_out/mc.err
DYCL_GEMM_NO_MC=1 timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/mc_off_$i.json 2>> gpurun_out/mc.err
done
for f in gpurun_out/mc_*.json; do python -c "import json,sys; l=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(l['ms_per_step'],2), {k:round(v,2) for k,v in l.get('kernel_ms_per_step',{}).items()})"; done
tail -3 gpurun_out/mc.err
timeout 1200 python -m pytest tests -m gpu -q -k "conv_kernel or cfg1 or mlp or cfg4 or s2s or seq2seq or caption or cfg5_resnet50_parity or cfg5_bench" 2>&1 | tail -2
