#!/bin/bash
# Round evidence: full GPU test suite, smoke, every workload through bench.py
mkdir -p gpurun_out
python -c "from paper_2307_04963_b200 import build as B; B.build()" > gpurun_out/build.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rs 2>&1 | tail -15 > gpurun_out/gputest_final.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.txt 2>&1
bash tools/bench_all.sh
tail -3 gpurun_out/gputest_final.txt; tail -1 gpurun_out/smoke_final.txt
for f in gpurun_out/bench_all.jsonl; do python -c "
import json
for line in open('$f'):
    l=json.loads(line); print(l.get('config',{}).get('workload','?')[:40], round(l.get('value',0),1), l.get('unit'), round(l.get('ms_per_step',0),3), (l.get('e2e') or {}).get('value'), l.get('clocks',{}).get('sm_mhz'))
"; done
