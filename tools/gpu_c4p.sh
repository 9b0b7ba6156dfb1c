#!/bin/bash
# cfg4: A/B (fused LN on/off), parity tests, ncu launch list of one batch (graph off) and
# --set full of one cross-attention launch and one fused-LN GEMM launch.
mkdir -p gpurun_out
rm -f gpurun_out/c4_*.json
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
for i in 1 2; do
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c4_new_$i.json 2> gpurun_out/c4.err
DYCL_S2S_FUSE_LN=0 timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c4_oldln_$i.json 2>> gpurun_out/c4.err
done
timeout 900 python -m pytest tests -m gpu -q -k "cfg4 or s2s or seq2seq" 2>&1 | tail -5 > gpurun_out/c4_tests.txt
for f in gpurun_out/c4_*.json; do python -c "import json,sys; l=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(l['ms_per_step'],2), {k:round(v,2) for k,v in l.get('kernel_ms_per_step',{}).items()})"; done
cat gpurun_out/c4_tests.txt
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
DYCL_S2S_GRAPH=0 timeout 900 ncu --metrics $M --clock-control none -k regex:k_ --csv \
   --log-file gpurun_out/c4_launches.csv python tools/s2s_probe.py 1024 1 > gpurun_out/c4_ncu.out 2>&1
DYCL_S2S_GRAPH=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_attn_cross_tma -s 20 -c 1 \
   -o gpurun_out/c4_xattn_full python tools/s2s_probe.py 1024 1 > gpurun_out/c4_full1.out 2>&1
DYCL_S2S_GRAPH=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tma -s 200 -c 6 \
   -o gpurun_out/c4_gemm_full python tools/s2s_probe.py 1024 1 > gpurun_out/c4_full2.out 2>&1
ls -la gpurun_out | tail -5
