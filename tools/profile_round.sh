#!/bin/bash
# Evidence pass for profiles/: launch list of one cfg2 step, per-launch DRAM bytes of the
# dominant kernel (k_block_fused), full ncu captures of the top kernels of cfg2 and cfg5.
# Skip counts are derived from the event-timed step (step_profile.py W: W warm runs, then
# the profiled run).  Run under gpurun; then: python tools/parse_profiles.py gpurun_out r01
set -x
mkdir -p gpurun_out
W=3
python tools/step_profile.py $W > gpurun_out/step_profile.json
read LPR NBLK <<< $(python - <<'P'
import json
p = json.load(open("gpurun_out/step_profile.json"))
print(len(p), sum(1 for q in p if q["kind"] == "block"))
P
)
# every launch of one warm step (ncu serialises + cold caches: compare SHARES)
ncu --metrics gpu__time_duration.sum --clock-control none -s $((W * LPR)) -c $LPR --csv \
    --log-file gpurun_out/launches.csv python tools/step_profile.py $W > /dev/null 2>&1
# DRAM bytes of every k_block_fused launch of one step
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:k_block_fused -s $((W * NBLK)) -c $NBLK --csv --log-file gpurun_out/block_dram.csv \
    python tools/step_profile.py $W > /dev/null 2>&1
# full captures: the first (stage-1, two-block) fused launch of the profiled step; a cfg-5 3x3 GEMM conv
ncu --set full --clock-control none --import-source on -k regex:k_block_fused -s $((W * NBLK)) -c 1 \
    -o gpurun_out/blk_full python tools/step_profile.py $W > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_conv_gemm -s 4 -c 2 \
    -o gpurun_out/gemm_full python tools/step_profile5.py 512 0 > /dev/null 2>&1
ls -la gpurun_out
