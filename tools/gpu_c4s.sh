#!/bin/bash
# cfg4: TMA-streamed self attention A/B (DYCL_XATTN_WARP=1 = per-warp form for both), parity tests
mkdir -p gpurun_out
rm -f gpurun_out/c4s_*.json
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
for i in 1 2; do
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c4s_new_$i.json 2> gpurun_out/c4s.err
DYCL_XATTN_WARP=1 timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c4s_old_$i.json 2>> gpurun_out/c4s.err
done
timeout 900 python -m pytest tests -m gpu -q -k "cfg4 or s2s or seq2seq" 2>&1 | tail -5 > gpurun_out/c4s_tests.txt
for f in gpurun_out/c4s_*.json; do python -c "import json,sys; l=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(l['ms_per_step'],2), {k:round(v,2) for k,v in l.get('kernel_ms_per_step',{}).items()})"; done
cat gpurun_out/c4s_tests.txt
timeout 600 python -m pytest tests/test_gpu.py -m gpu -q -s -k "zero_copy" 2>&1 | tail -4 >> gpurun_out/c4s_tests.txt; tail -4 gpurun_out/c4s_tests.txt
