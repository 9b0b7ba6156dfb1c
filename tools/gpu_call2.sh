#!/bin/bash
# One gpurun call: GPU tests (verbose cfg4 parity) + cfg4 bench + launch list of one cfg4 batch.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -25 > gpurun_out/pytest_tail.txt
tail -3 gpurun_out/pytest_tail.txt
timeout 300 python -m pytest tests/test_gpu.py -m gpu -q -s -k cfg4 2>&1 | grep -i "cfg4\|passed\|failed" | head -10
timeout 300 python bench.py --config 1 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench1.json 2> gpurun_out/bench1.err; python -c "import json; d=json.load(open('gpurun_out/bench1.json')); print('bench1', d['ms_per_step'])"
timeout 300 python bench.py --config 4 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench4.json 2> gpurun_out/bench4.err
python -c "import json; d=json.load(open('gpurun_out/bench4.json')); print('bench4', d['ms_per_step'], d['value'], d['e2e']['value'], d['config'].get('decisions_rank0'), d.get('kernel_ms_per_step'))"
if [ -n "$LAUNCHES" ]; then timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s2s_launches.csv python tools/s2s_probe.py 1024 1 > gpurun_out/s2s_probe.log 2>&1; fi
