#!/bin/bash
# cfg5: ncu launch list (+ DRAM bytes) of one 2048-row chunk, run launch by launch (graph off)
mkdir -p gpurun_out
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active
DYCL_GRAPH=0 timeout 900 ncu --metrics $M --clock-control none -k regex:k_ --csv \
   --log-file gpurun_out/c5_launches.csv python tools/ncu_chunk.py 5 2048 > gpurun_out/c5_ncu.out 2>&1
python tools/launch_list.py gpurun_out/c5_launches.csv | head -20
