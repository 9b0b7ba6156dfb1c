#!/bin/bash
# Dev pass: build, targeted gpu tests, cfg5 per-launch profile.
mkdir -p gpurun_out
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_rnn.py tests/test_abi.py -q -x 2>&1 | tail -15 > gpurun_out/dev_rnn.txt
timeout 1500 python -m pytest tests/test_gpu.py tests/test_gpu_edge.py tests/test_gpu_multi.py -m gpu -q -k "cfg5 or cfg4_seq2seq_parity or rebalance or shards" 2>&1 | tail -25 > gpurun_out/dev_tests.txt
timeout 300 python tools/step_profile5.py 2048 2 > gpurun_out/prof5.json 2> gpurun_out/prof5.err
tail -3 gpurun_out/dev_rnn.txt; tail -3 gpurun_out/dev_tests.txt
