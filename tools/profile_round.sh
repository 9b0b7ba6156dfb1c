#!/bin/bash
# Evidence pass for profiles/: launch list, per-launch DRAM bytes of the conv kernel,
# one full ncu capture of a stage-1 conv launch, and the library's own per-launch timing.
set -x
mkdir -p gpurun_out
python tools/step_profile.py 3 > gpurun_out/step_profile.json
# every launch of one warm step (ncu serialises + cold caches: compare SHARES)
ncu --metrics gpu__time_duration.sum --clock-control none -s 240 -c 80 --csv \
    --log-file gpurun_out/launches.csv python tools/step_profile.py 3 > /dev/null 2>&1
# DRAM bytes of every conv launch of one step
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:k_conv -s 165 -c 55 --csv --log-file gpurun_out/conv_dram.csv python tools/step_profile.py 3 > /dev/null 2>&1
# one full capture: stem(0), conv1(1), conv2(2) of the first block of the measured step
ncu --set full --clock-control none --import-source on -k regex:k_conv_tma -s 166 -c 2 \
    -o gpurun_out/conv_full python tools/step_profile.py 3 > /dev/null 2>&1
ls -la gpurun_out
