#!/bin/bash
# cfg5 --set full: k_cast_s4d, k_conv_gemm #0 (block-1 conv1), #3 (stage-1 conv3 + residual), #5 (same + fused GAP)
mkdir -p gpurun_out
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
DYCL_GRAPH=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cast_s4d -c 1 \
   -o gpurun_out/c5_cast python tools/ncu_chunk.py 5 2048 > gpurun_out/c5_cast.out 2>&1
for s in 0 3 5; do
DYCL_GRAPH=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_conv_gemm -s $s -c 1 \
   -o gpurun_out/c5_conv2_s$s python tools/ncu_chunk.py 5 2048 > gpurun_out/c5_full2_s$s.out 2>&1
done
ls -la gpurun_out/*.ncu-rep
