#!/bin/bash
# Round-2 evidence pass (run under gpurun; then: python tools/parse_r02.py):
#  cfg5 (headline): ncu launch list + DRAM bytes of every launch of one 2048-row chunk, run launch by
#  launch (DYCL_GRAPH=0); --set full of two stage-1 k_conv_gemm launches (conv2 3x3, conv3 1x1+residual)
#  cfg2: launch list + DRAM of one step; --set full of the first k_block_fused launch
#  cfg4: launch list of one 1024-sequence batch (graph off)
#  sanitizers: racecheck / synccheck on tests that run k_block_fused, k_conv_gemm and the s2s chain
set -x
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
DYCL_GRAPH=0 timeout 900 ncu --metrics $M --clock-control none -k regex:k_ --csv \
   --log-file gpurun_out/c5_launches.csv python tools/ncu_chunk.py 5 2048 > gpurun_out/c5_ncu.out 2>&1
DYCL_GRAPH=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_conv_gemm -s 4 -c 2 \
   -o gpurun_out/c5_conv_full python tools/ncu_chunk.py 5 2048 > gpurun_out/c5_full.out 2>&1
DYCL_GRAPH=0 timeout 900 ncu --metrics $M --clock-control none -k regex:k_ --csv \
   --log-file gpurun_out/c2_launches.csv python tools/ncu_chunk.py 2 4096 > gpurun_out/c2_ncu.out 2>&1
DYCL_GRAPH=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_block_fused -c 1 \
   -o gpurun_out/c2_block_full python tools/ncu_chunk.py 2 4096 > gpurun_out/c2_full.out 2>&1
DYCL_S2S_GRAPH=0 timeout 900 ncu --metrics $M --clock-control none -k regex:k_ --csv \
   --log-file gpurun_out/c4_launches.csv python tools/s2s_probe.py 1024 1 > gpurun_out/c4_ncu.out 2>&1
for tool in racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --log-file gpurun_out/${tool}_r02.log \
    python -m pytest -m gpu -q -x "tests/test_gpu.py::test_cfg2_sdn_parity[1]" "tests/test_gpu.py::test_cfg4_seq2seq_parity[1]" \
      "tests/test_gpu.py::test_cfg1_mlp_parity" tests/test_gpu.py::test_conv_gemm_nhwc_matches_oracle_conv \
    > gpurun_out/${tool}_r02.out 2>&1
done
timeout 1200 compute-sanitizer --tool memcheck --log-file gpurun_out/memcheck_r02.log \
  python -m pytest -m gpu -q -x "tests/test_gpu.py::test_cfg2_sdn_parity[203]" "tests/test_gpu_rnn.py::test_cfg3r_rnn_skipnet_parity" \
    tests/test_gpu.py::test_cfg5_resnet50_parity "tests/test_gpu.py::test_cfg4_seq2seq_parity[5]" tests/test_gpu.py::test_cfg3_skipnet_parity \
  > gpurun_out/memcheck_r02.out 2>&1
ls -la gpurun_out | tail -30
