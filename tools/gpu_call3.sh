#!/bin/bash
# smoke() + compute-sanitizer memcheck / racecheck on the config-4 parity tests (PDL chain, new kernels)
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 1200 compute-sanitizer --tool memcheck --log-file gpurun_out/memcheck_s2s.log python -m pytest tests/test_gpu.py -m gpu -x -q -k "cfg4_seq2seq_parity or cfg1" 2>&1 | tail -2
tail -2 gpurun_out/memcheck_s2s.log
timeout 1200 compute-sanitizer --tool racecheck --log-file gpurun_out/racecheck_s2s.log python -m pytest tests/test_gpu.py -m gpu -x -q -k "cfg4_seq2seq_parity and 8" 2>&1 | tail -2
tail -2 gpurun_out/racecheck_s2s.log
