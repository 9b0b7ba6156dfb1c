#!/bin/bash
# cfg4: encoder attention Q/K by TMA + cheaper fused argmax; bench x2, cfg4 + caption tests, launch list
mkdir -p gpurun_out
rm -f gpurun_out/c4e_*.json
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -rf 2>&1 | grep -E "passed|failed|FAILED" > gpurun_out/multi_tests.txt
for i in 1 2; do
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c4e_$i.json 2> gpurun_out/c4e.err
done
timeout 900 python -m pytest tests -m gpu -q -k "cfg4 or s2s or seq2seq or caption or cap" 2>&1 | tail -3 > gpurun_out/c4e_tests.txt
for f in gpurun_out/c4e_*.json; do python -c "import json,sys; l=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(l['ms_per_step'],2), {k:round(v,2) for k,v in l.get('kernel_ms_per_step',{}).items()})"; done
cat gpurun_out/c4e_tests.txt
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
DYCL_S2S_GRAPH=0 timeout 900 ncu --metrics $M --clock-control none -k regex:k_ --csv \
   --log-file gpurun_out/c4_launches4.csv python tools/s2s_probe.py 1024 1 > gpurun_out/c4_ncu4.out 2>&1
python tools/launch_list.py gpurun_out/c4_launches4.csv | head -12
cat gpurun_out/multi_tests.txt
