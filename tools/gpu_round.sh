#!/bin/bash
# One GPU pass: gpu tests, smoke, bench (default cfg5 + cfg2). Outputs under gpurun_out/.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 1500 python -m pytest tests -m gpu -x -q -rs 2>&1 | tail -30 > gpurun_out/gputest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 600 python bench.py --config 2 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
tail -3 gpurun_out/gputest.txt; tail -1 gpurun_out/smoke.txt; tail -c 3000 gpurun_out/bench_c5.json; tail -c 1500 gpurun_out/bench_c2.json
