#!/bin/bash
# sanitizers on the kernels added in round 2 (halo conv, caption decoder, device rebalancing) + a cfg5 profile
mkdir -p gpurun_out
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
: > gpurun_out/sanitizers_r02b.txt
for tool in memcheck synccheck racecheck; do
  for t in "tests/test_gpu.py::test_conv_gemm_nhwc_matches_oracle_conv" "tests/test_gpu_caption.py::test_caption_parity" \
           "tests/test_gpu_multi.py::test_cfg2_rebalance_on_equals_off" "tests/test_gpu_rnn.py::test_cfg3r_rnn_skipnet_parity"; do
    tag=$(echo $t | sed 's/.*:://')
    timeout 900 compute-sanitizer --tool $tool --log-file gpurun_out/${tool}_${tag}.log python -m pytest -m gpu -q -x "$t" > gpurun_out/${tool}_${tag}.out 2>&1
    echo "$tool $t rc=$? $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' gpurun_out/${tool}_${tag}.log | tail -1) $(tail -1 gpurun_out/${tool}_${tag}.out)" >> gpurun_out/sanitizers_r02b.txt
  done
done
timeout 300 python tools/step_profile5.py 2048 2 > gpurun_out/prof5.json 2> gpurun_out/prof5.err
cat gpurun_out/sanitizers_r02b.txt
