ncu --set full --clock-control none --import-source on -k regex:k_conv_tma -s 61 -c 1 -o gpurun_out/conv64_full python tools/step_profile.py 3 > gpurun_out/ncu1.log 2>&1
tail -3 gpurun_out/ncu1.log
