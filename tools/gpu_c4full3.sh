#!/bin/bash
# --set full of the final decode kernels: the DSMEM-LayerNorm cluster GEMM (k_gemm_tma<64>) and k_attn_tma
mkdir -p gpurun_out
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
DYCL_S2S_GRAPH=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tma -s 300 -c 6 \
   -o gpurun_out/c4f_gemm python tools/s2s_probe.py 1024 1 > gpurun_out/c4f1.out 2>&1
DYCL_S2S_GRAPH=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_attn_tma -s 40 -c 2 \
   -o gpurun_out/c4f_attn python tools/s2s_probe.py 1024 1 > gpurun_out/c4f2.out 2>&1
ls -la gpurun_out/c4f_*.ncu-rep
