#!/bin/bash
# Final evidence: full GPU test suite, smoke, every workload through bench.py, launch lists cfg4 / cfg5
mkdir -p gpurun_out
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rs 2>&1 | tail -15 > gpurun_out/gputest_final.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.txt 2>&1
bash tools/bench_all.sh
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
DYCL_S2S_GRAPH=0 timeout 900 ncu --metrics $M --clock-control none -k regex:k_ --csv \
   --log-file gpurun_out/c4_launches_final.csv python tools/s2s_probe.py 1024 1 > gpurun_out/c4_ncu_final.out 2>&1
DYCL_GRAPH=0 timeout 900 ncu --metrics $M,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_ --csv \
   --log-file gpurun_out/c5_launches_final.csv python tools/ncu_chunk.py 5 2048 > gpurun_out/c5_ncu_final.out 2>&1
tail -3 gpurun_out/gputest_final.txt; tail -1 gpurun_out/smoke_final.txt
python -c "
import json
for line in open('gpurun_out/bench_all.jsonl'):
    l=json.loads(line); print(l.get('config',{}).get('workload','?')[:40], round(l.get('value',0),1), l.get('unit'), round(l.get('ms_per_step',0),3), (l.get('e2e') or {}).get('value'), l.get('clocks',{}).get('sm_mhz'))
"
python tools/launch_list.py gpurun_out/c4_launches_final.csv | tail -1
python tools/launch_list.py gpurun_out/c5_launches_final.csv | tail -1
