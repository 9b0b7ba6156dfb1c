#!/bin/bash
# sanitizers on the round-2-session kernels: cfg4 (k_attn_tma pre-wait ring, DSMEM LayerNorm
# cluster GEMM, pre-issued weight boxes), cfg5 conv (GAP transpose-reduce), device rebalancing
mkdir -p gpurun_out
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
for tool in memcheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --log-file gpurun_out/${tool}_s3.log \
    python -m pytest -m gpu -q -x "tests/test_gpu.py::test_cfg4_seq2seq_parity[5]" "tests/test_gpu.py::test_cfg1_mlp_parity" \
    > gpurun_out/${tool}_s3.out 2>&1
  echo "$tool: $(tail -1 gpurun_out/${tool}_s3.out) | $(grep -E 'ERROR SUMMARY|error' gpurun_out/${tool}_s3.log | tail -2 | tr '\n' ' ')"
done
timeout 1200 compute-sanitizer --tool racecheck --log-file gpurun_out/racecheck_s3.log \
  python -m pytest -m gpu -q -x "tests/test_gpu.py::test_cfg4_seq2seq_parity[1]" > gpurun_out/racecheck_s3.out 2>&1
echo "racecheck: $(tail -1 gpurun_out/racecheck_s3.out) | $(grep -E 'RACECHECK SUMMARY|hazard' gpurun_out/racecheck_s3.log | tail -2 | tr '\n' ' ')"
