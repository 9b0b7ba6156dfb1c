#!/bin/bash
# One gpurun call: GPU tests + bench of configs 1, 2, 4 (PDL on / off for 1 and 2).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -25 > gpurun_out/pytest_tail.txt
tail -3 gpurun_out/pytest_tail.txt
for c in 1 2; do
  DYCL_PDL=0 timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench${c}_nopdl.json 2> gpurun_out/bench${c}_nopdl.err
  timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench${c}.json 2> gpurun_out/bench${c}.err
done
timeout 300 python bench.py --config 4 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench4.json 2> gpurun_out/bench4.err
for f in gpurun_out/bench1_nopdl.json gpurun_out/bench1.json gpurun_out/bench2_nopdl.json gpurun_out/bench2.json gpurun_out/bench4.json; do
python -c "import json; d=json.load(open('$f')); print('$f', round(d['ms_per_step'],4), round(d['value']), round(d['e2e']['value']), d['config'].get('decisions_rank0'))"; done
