#!/bin/bash
# s4d cast with a TMA tensor store: cfg5 parity + bench x2 + ncu DRAM bytes of the cast
mkdir -p gpurun_out
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu.py tests/test_gpu_edge.py -m gpu -q -x -k "cfg5" 2>&1 | tail -2
for i in 1 2; do
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/cast_$i.json 2> gpurun_out/cast.err
done
for f in gpurun_out/cast_*.json; do python -c "import json,sys; l=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(l['ms_per_step'],2), l['clocks']['sm_mhz'], {k:round(v,2) for k,v in l.get('kernel_ms_per_step',{}).items()})"; done
DYCL_GRAPH=0 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum --clock-control none -k regex:k_cast_s4d -c 1 python tools/ncu_chunk.py 5 2048 2>&1 | grep -E "duration|dram__|lts__" 
