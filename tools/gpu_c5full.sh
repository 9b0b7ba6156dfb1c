#!/bin/bash
# cfg5: ncu --set full of three k_conv_gemm launches of one 2048-row chunk (graph off):
#  #0 block-1 conv1 (1x1 64->64 @56x56), #5 stage-1 last conv3 + residual + fused GAP, #8 stage-2 conv3 + zero-copy projection
mkdir -p gpurun_out
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
for s in 0 5 8; do
DYCL_GRAPH=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_conv_gemm -s $s -c 1 \
   -o gpurun_out/c5_conv_s$s python tools/ncu_chunk.py 5 2048 > gpurun_out/c5_full_s$s.out 2>&1
done
ls -la gpurun_out/*.ncu-rep
