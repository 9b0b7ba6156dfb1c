#!/bin/bash
# Evidence pass for profiles/: launch list, per-launch DRAM bytes of the conv-class kernels
# (fused blocks, implicit-GEMM convs, dense GEMMs), one full ncu capture of the top fused-block
# and conv launches, and the library's own per-launch timing.  Skip counts are derived from
# the event-timed step (step_profile.py W: W warm runs, then the profiled run).
set -x
mkdir -p gpurun_out
W=3
python tools/step_profile.py $W > gpurun_out/step_profile.json
read LPR NCONV FIRST_BLK FIRST_CONV <<< $(python - <<'EOF'
import json
p = json.load(open("gpurun_out/step_profile.json"))
conv = [i for i, q in enumerate(p) if q["kind"] == "conv"]
print(len(p), len(conv), 0, 0)
EOF
)
RE='regex:k_block_fused|k_conv|k_gemm'
# every launch of one warm step (ncu serialises + cold caches: compare SHARES)
ncu --metrics gpu__time_duration.sum --clock-control none -s $((W * LPR)) -c $LPR --csv \
    --log-file gpurun_out/launches.csv python tools/step_profile.py $W > /dev/null 2>&1
# DRAM bytes of every conv-class launch of one step
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k "$RE" -s $((W * NCONV)) -c $NCONV --csv --log-file gpurun_out/conv_dram.csv \
    python tools/step_profile.py $W > /dev/null 2>&1
# full captures: the first stage-1 fused block launch and the first unfused 3x3 conv launch of the step
ncu --set full --clock-control none --import-source on -k regex:k_block_fused -s 8 -c 1 \
    -o gpurun_out/blk_full python tools/step_profile.py $W > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_conv_tma -s 8 -c 1 \
    -o gpurun_out/conv_full python tools/step_profile.py $W > /dev/null 2>&1
ls -la gpurun_out
