#!/bin/bash
# cfg5: conv kernel tests + cfg5 parity/zero-copy tests + 2 bench runs + launch list of one chunk
mkdir -p gpurun_out
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu.py tests/test_gpu_multi.py tests/test_gpu_edge.py -m gpu -q -x -k "nhwc or cfg5 or zero_copy" 2>&1 | tail -3 > gpurun_out/c5ab_tests.txt
for i in 1 2; do
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c5ab_$i.json 2> gpurun_out/c5ab.err
done
for f in gpurun_out/c5ab_*.json; do python -c "import json,sys; l=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(l['ms_per_step'],2), l['clocks']['sm_mhz'], {k:round(v,2) for k,v in l.get('kernel_ms_per_step',{}).items()})"; done
cat gpurun_out/c5ab_tests.txt
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active
DYCL_GRAPH=0 timeout 900 ncu --metrics $M --clock-control none -k regex:k_ --csv \
   --log-file gpurun_out/c5_launches2.csv python tools/ncu_chunk.py 5 2048 > gpurun_out/c5_ncu2.out 2>&1
python tools/launch_list.py gpurun_out/c5_launches2.csv | tail -1
