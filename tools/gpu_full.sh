#!/bin/bash
# full GPU test suite + smoke + bench (cfg5 default, cfg2) -- a round checkpoint
mkdir -p gpurun_out
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rs 2>&1 | tail -20 > gpurun_out/gputest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 600 python bench.py --config 2 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
tail -3 gpurun_out/gputest.txt; tail -1 gpurun_out/smoke.txt
