#!/bin/bash
# cfg4: decode weights in a persisting L2 window on/off; cfg4 tests
mkdir -p gpurun_out
rm -f gpurun_out/c4l2_*.json
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
python -c "
import torch; p=torch.cuda.get_device_properties(0); print('L2', p.L2_cache_size, 'persist max', getattr(p,'persisting_l2_cache_max_size',None))" > gpurun_out/l2.txt 2>&1
for i in 1 2; do
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c4l2_on_$i.json 2> gpurun_out/c4l2.err
DYCL_S2S_L2PERSIST=0 timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c4l2_off_$i.json 2>> gpurun_out/c4l2.err
done
timeout 900 python -m pytest tests -m gpu -q -k "cfg4 or s2s or seq2seq" 2>&1 | tail -3 > gpurun_out/c4l2_tests.txt
for f in gpurun_out/c4l2_*.json; do python -c "import json,sys; l=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(l['ms_per_step'],2), {k:round(v,2) for k,v in l.get('kernel_ms_per_step',{}).items()})"; done
cat gpurun_out/c4l2_tests.txt gpurun_out/l2.txt; tail -3 gpurun_out/c4l2.err
