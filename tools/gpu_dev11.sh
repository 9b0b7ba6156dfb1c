#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu.py tests/test_gpu_edge.py tests/test_gpu_rnn.py -m gpu -q -x 2>&1 | tail -5 > gpurun_out/dev_tests.txt
cat gpurun_out/dev_tests.txt | tail -3
for c in 2 3 1 5; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
  python -c "import json;d=json.loads(open('gpurun_out/bench_c$c.json').read().strip().splitlines()[-1]);print($c, d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
done
