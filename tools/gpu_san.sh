#!/bin/bash
# sanitizers (per-target, bounded) + RQ3 ablation + cfg2 block tests after the xb_empty change
mkdir -p gpurun_out
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu.py -m gpu -q -x -k "cfg2 or cfg3 or zero_copy or in_place or graph_replay or permutation" 2>&1 | tail -3 > gpurun_out/dev_tests.txt
for tool in synccheck racecheck; do
  for t in "tests/test_gpu.py::test_cfg2_sdn_parity[1]" "tests/test_gpu.py::test_cfg1_mlp_parity" \
           "tests/test_gpu.py::test_cfg4_seq2seq_parity[1]" "tests/test_gpu.py::test_conv_gemm_nhwc_matches_oracle_conv" \
           "tests/test_gpu_rnn.py::test_cfg3r_forced_gates"; do
    tag=$(echo $t | sed 's/.*:://; s/\[.*//')
    timeout 900 compute-sanitizer --tool $tool --log-file gpurun_out/${tool}_${tag}.log python -m pytest -m gpu -q -x "$t" > gpurun_out/${tool}_${tag}.out 2>&1
    echo "$tool $t rc=$? $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY\|hazard' gpurun_out/${tool}_${tag}.log | tail -1) $(tail -1 gpurun_out/${tool}_${tag}.out)" >> gpurun_out/sanitizers_r02.txt
  done
done
bash tools/rq3_ablation.sh > gpurun_out/rq3.log 2>&1
cat gpurun_out/dev_tests.txt gpurun_out/sanitizers_r02.txt
