#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/emb_*.json
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
for i in 1 2; do
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/emb_$i.json 2> gpurun_out/ring.err
done
for f in gpurun_out/emb_*.json; do python -c "import json,sys; l=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(l['ms_per_step'],2), {k:round(v,2) for k,v in l.get('kernel_ms_per_step',{}).items()})"; done
tail -3 gpurun_out/ring.err
timeout 900 python -m pytest tests -m gpu -q -k "cfg4 or s2s or seq2seq" 2>&1 | tail -2
